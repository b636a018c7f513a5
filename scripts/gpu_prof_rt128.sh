mkdir -p gpurun_out/rt128
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cos_.*_rt -c 2 -o gpurun_out/rt128/prof -f python bench.py --workload long4k_d128 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/rt128/log.txt 2>&1
tail -2 gpurun_out/rt128/log.txt
