# Round-2 check b: GPU tests, bench with kernel stamps, bf16 MMA probe, ML-1M phase trace.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=20 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
./scripts/dev/mma_probe_bf16 > gpurun_out/probe_bf16.txt 2>&1
bash scripts/gpu_trace.sh > gpurun_out/trace.txt 2>&1
tail -3 gpurun_out/pytest_gpu.log; grep FAILED gpurun_out/pytest_gpu.log | head -20
python -c "
import json; d=json.load(open('gpurun_out/bench.json')); k=d.get('kernels',{}); print('value=%.4g'%d['value'], 'ms=%.4f'%d['ms_per_step'], k, d['roofline'].get('ops_sum_over_step'), 'e2e', d.get('e2e',{}).get('value'), d.get('clocks')); print(d['steady_state'])"
tail -3 gpurun_out/bench.err; cat gpurun_out/probe_bf16.txt; cat gpurun_out/trace.txt
