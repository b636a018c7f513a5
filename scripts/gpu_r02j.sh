# Session re-entry check: GPU tests, smoke, default bench + reference arm.
mkdir -p gpurun_out/r02j
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r02j/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02j/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02j/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02j/smoke.log
timeout 600 python bench.py > gpurun_out/r02j/bench.json 2> gpurun_out/r02j/bench.err
timeout 400 python bench.py --impl reference > gpurun_out/r02j/bench_ref.json 2>> gpurun_out/r02j/bench.err
tail -5 gpurun_out/r02j/pytest_gpu.log; tail -2 gpurun_out/r02j/smoke.log
cat gpurun_out/r02j/bench.json | head -c 3000; echo; cat gpurun_out/r02j/bench_ref.json | head -c 1500
