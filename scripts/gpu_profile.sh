# Profiles only (kept under the 64 MiB gpurun_out cap): launch lists + one full ncu capture.
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_ml1m.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2> gpurun_out/prof.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:d32 -c 8 --csv --log-file gpurun_out/launches_ml20m.csv python bench.py --workload ml20m --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>> gpurun_out/prof.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:d32 -s 2 -c 2 -o gpurun_out/prof_ml20m -f python bench.py --workload ml20m --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>> gpurun_out/prof.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:d32 -s 4 -c 4 --csv --log-file gpurun_out/metrics_ml1m.csv python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu > /dev/null 2>> gpurun_out/prof.err
ls -la gpurun_out; tail -3 gpurun_out/prof.err
