# ncu of the register-tiled d_h 64/128 kernels (one launch each of fwd and bwd) at long4k_d64
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:_rt -s 2 -c 2 -o gpurun_out/prof_rt_d64 -f python bench.py --workload long4k_d64 --steps 1 --warmup 1 --no-e2e --no-cpu --graph off > gpurun_out/prof_rt.log 2>&1
tail -3 gpurun_out/prof_rt.log
