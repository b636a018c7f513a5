# bf16 d_h=32 on tcgen05 (paired rows): parity, then bench vs the register-tiled kernels
mkdir -p gpurun_out/pair
timeout 900 python -m pytest tests/test_gpu_tcb.py -q -p no:cacheprovider -x > gpurun_out/pair/pytest_tcb.log 2>&1; echo "rc=$?" >> gpurun_out/pair/pytest_tcb.log
tail -15 gpurun_out/pair/pytest_tcb.log
for n in 512 4096 16384; do
  w=sw_n${n}_d32_bf16
  timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/pair/$w.json 2>gpurun_out/pair/$w.err
  COTTEN_NO_TCB_PAIR=1 timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/pair/${w}_rt.json 2>>gpurun_out/pair/$w.err
  for f in gpurun_out/pair/$w.json gpurun_out/pair/${w}_rt.json; do python -c "
import json,sys
try:
  d=json.load(open('$f')); k=d['kernels']; print('$f', 'value=%.4g'%d['value'], 'fwd %.3f bwd %.3f step %.3f'%(k['fwd_frac'],k['bwd_frac'],k['step_frac']), d['run']['kernel_path'], d['clocks']['sm_mhz'])
except Exception as e: print('$f ERR', e)
"; done
  tail -2 gpurun_out/pair/$w.err
done
