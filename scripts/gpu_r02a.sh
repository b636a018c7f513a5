# Round-2 check: GPU tests (incl. the multi-unit schedule and boundary tests),
# smoke, both bench arms, compute-sanitizer on every kernel path.
mkdir -p gpurun_out/san
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.csv 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 400 python bench.py --impl reference > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
timeout 400 python bench.py --no-steady --no-cpu --no-e2e > gpurun_out/bench_noev.json 2>> gpurun_out/bench.err
for p in tc tclong d32 rt64 rt128 rtbf16 generic; do
  for tool in memcheck racecheck synccheck; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_case.py $p > gpurun_out/san/${tool}_$p.log 2>&1; echo "rc=$?" >> gpurun_out/san/${tool}_$p.log
  done
done
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log
for f in bench bench_noev; do python -c "
import json; d=json.load(open('gpurun_out/$f.json')); k=d.get('kernels',{}); print('$f', 'value=%.4g'%d['value'], 'ms=%.4f'%d['ms_per_step'], k, 'e2e', d.get('e2e',{}).get('value'), 'cpu', d.get('cpu_baseline',{}).get('value'), 'launches', d.get('gpu_launches'), d.get('clocks'))" 2>&1 | tail -1; done
cut -c1-300 gpurun_out/bench_ref.json; tail -3 gpurun_out/bench.err
grep -H "ERROR SUMMARY\|rc=" gpurun_out/san/*.log
