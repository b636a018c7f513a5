# tcgen05 bring-up: parity tests for the d32 paths first, then bench both paths.
mkdir -p gpurun_out
timeout 300 python scripts/dev/err_table.py > gpurun_out/err_table.txt 2>&1; cat gpurun_out/err_table.txt | tail -12
timeout 300 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
for path in tcgen05 fp32pipe; do
for w in ml1m ml20m beauty; do
timeout 300 python bench.py --workload $w --path $path --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_${w}_${path}.json 2>> gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench_${w}_${path}.json')); k=d['kernels']; print('$w $path', 'value=%.4g'%d['value'], 'ms=%.4f'%d['ms_per_step'], 'fwd %.1fus %.3f'%(k['fwd_us'],k['fwd_frac']), 'bwd %.1fus %.3f'%(k['bwd_us'],k['bwd_frac']), 'step %.3f'%k['step_frac'])" 2>&1 | tail -1
done; done
tail -5 gpurun_out/bench.err
bash scripts/gpu_trace.sh
