mkdir -p gpurun_out/beautyprof
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tcf_kernel -c 2 -o gpurun_out/beautyprof/prof -f python bench.py --workload beauty --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/beautyprof/log.txt 2>&1
tail -2 gpurun_out/beautyprof/log.txt
