# Round-2 ML-1M diagnosis: phase trace (trace build) + ncu full capture of the
# ML-1M tcgen05 fwd and bwd + the launch list of the default bench command.
mkdir -p gpurun_out
bash scripts/gpu_trace.sh > gpurun_out/trace.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_ml1m.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-steady > /dev/null 2> gpurun_out/prof.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_kernel -s 4 -c 2 -o gpurun_out/prof_tc_ml1m -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-steady --graph off > /dev/null 2>> gpurun_out/prof.err
cat gpurun_out/trace.txt; tail -3 gpurun_out/prof.err; ls -la gpurun_out
