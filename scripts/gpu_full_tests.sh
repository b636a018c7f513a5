# Full GPU test suite + smoke
mkdir -p gpurun_out/full
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/full/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/full/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/full/smoke.log
tail -8 gpurun_out/full/pytest_gpu.log; tail -2 gpurun_out/full/smoke.log
for n in 1024 2048 8192 16384; do
  w=sw_n${n}_d64_f32
  timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/full/$w.json 2>gpurun_out/full/$w.err
done
