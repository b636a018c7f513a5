# ncu --set full with source of the fp32 tcgen05 kernels at ML-20M (one launch each)
mkdir -p gpurun_out/r02k
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_kernel -s 2 -c 2 -o gpurun_out/r02k/prof_tc_ml20m -f python bench.py --workload ml20m --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r02k/prof_tc.log 2>&1
tail -3 gpurun_out/r02k/prof_tc.log
ls -la gpurun_out/r02k/
