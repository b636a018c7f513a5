# Launch list (per-kernel durations) of the encoder training step
mkdir -p gpurun_out/enc
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/enc/launches.csv python bench.py --encoder-only --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/enc/b.log 2>&1
python scripts/launch_table.py gpurun_out/enc/launches.csv
wc -l gpurun_out/enc/launches.csv
