# ncu --set full (with source) of the tcgen05 kernels: fp32 d_h=64 (tcf) at N=4096, fp32 d_h=32 (tc) at ML-20M
mkdir -p gpurun_out/r02m
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tcf_kernel -c 2 -o gpurun_out/r02m/prof_tcf -f python bench.py --workload sw_n4096_d64_f32 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r02m/prof_tcf.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_kernel -s 2 -c 2 -o gpurun_out/r02m/prof_tc_ml20m -f python bench.py --workload ml20m --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r02m/prof_tc.log 2>&1
tail -2 gpurun_out/r02m/prof_tcf.log gpurun_out/r02m/prof_tc.log
ls -la gpurun_out/r02m/
