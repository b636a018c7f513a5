# last full check: GPU suite, smoke, default bench line, reference arm
mkdir -p gpurun_out/last
timeout 2400 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/last/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/last/pytest_gpu.log
tail -3 gpurun_out/last/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/last/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/last/smoke.log; tail -2 gpurun_out/last/smoke.log
timeout 900 python bench.py > gpurun_out/last/bench.json 2> gpurun_out/last/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/last/bench_ref.json 2>> gpurun_out/last/bench.err
python -c "
import json; d=json.load(open('gpurun_out/last/bench.json')); k=d['kernels']; print('default', d['value'], 'fwd %.3f bwd %.3f step %.3f' % (k['fwd_frac'], k['bwd_frac'], k['step_frac']), 'e2e', d['e2e']['value'], d['e2e'].get('repeats_seq_per_s'), 'cpu', d['cpu_baseline']['value'], d['clocks'])
r=json.load(open('gpurun_out/last/bench_ref.json')); print('ref', r['value'])"
