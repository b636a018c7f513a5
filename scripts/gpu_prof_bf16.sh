# ncu --set full of the bf16 tensor-core kernels at config #5 points: tcb paired rows (d_h 32) and tch (d_h 128)
mkdir -p gpurun_out/pb
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cos_.*_tcb -c 2 -o gpurun_out/pb/tcb_pair python bench.py --workload sw_n4096_d32_bf16 --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cos_.*_tch -c 2 -o gpurun_out/pb/tch python bench.py --workload sw_n4096_d128_bf16 --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1
ls -la gpurun_out/pb
