# bf16 tcgen05 kernels: parity + A/B bench vs the FP32-pipe kernels
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tcb.py -q -p no:cacheprovider -x > gpurun_out/pytest_tcb.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tcb.log
tail -25 gpurun_out/pytest_tcb.log
for w in long4k_d64_bf16; do
  timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/b_$w.json 2>gpurun_out/b_$w.err
  COTTEN_NO_TCB=1 timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/b_${w}_rt.json 2>>gpurun_out/b_$w.err
  python -c "
import json
for f in ('gpurun_out/b_$w.json','gpurun_out/b_${w}_rt.json'):
  try:
    d=json.load(open(f)); print(f, 'value=%.4g'%d['value'], d['kernels'], d['run']['kernel_path'])
  except Exception as e: print(f, 'ERR', e)
"
  tail -3 gpurun_out/b_$w.err
done
