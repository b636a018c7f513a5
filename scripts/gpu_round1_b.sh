set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --workload ml20m --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_ml20m.json 2>> gpurun_out/bench.err
timeout 300 python bench.py --workload beauty --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_beauty.json 2>> gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>> gpurun_out/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cos_ -s 4 -c 2 -o gpurun_out/prof_ml20m python bench.py --workload ml20m --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>> gpurun_out/bench.err
tail -5 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log gpurun_out/bench.json gpurun_out/bench_ml20m.json gpurun_out/bench_beauty.json
