# Encoder training step bench line + its ncu launch list (kernel shares)
mkdir -p gpurun_out
timeout 600 python bench.py --encoder-only --steps 10 --warmup 3 > gpurun_out/bench_enc.json 2> gpurun_out/bench_enc.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_enc.csv python bench.py --encoder-only --steps 1 --warmup 3 --no-cpu > /dev/null 2>> gpurun_out/bench_enc.err
tail -5 gpurun_out/bench_enc.err; cat gpurun_out/bench_enc.json | head -c 3000
