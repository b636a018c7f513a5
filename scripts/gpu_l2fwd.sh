# forward L2 prefetch at long N (default on for C >= 8) vs off
mkdir -p gpurun_out/l2fwd
timeout 900 python -m pytest tests/test_gpu_tcf.py tests/test_gpu_tcb.py tests/test_gpu_schedule.py -q -p no:cacheprovider -x > gpurun_out/l2fwd/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/l2fwd/pytest.log
tail -2 gpurun_out/l2fwd/pytest.log
for w in sw_n1024_d32_f32 sw_n4096_d32_f32 sw_n16384_d32_f32 sw_n4096_d64_f32 sw_n4096_d64_bf16 sw_n4096_d32_bf16; do
  for pf in default 0; do
    if [ $pf = default ]; then unset COTTEN_L2_AHEAD; else export COTTEN_L2_AHEAD=0; fi
    timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/l2fwd/${w}_$pf.json 2>>gpurun_out/l2fwd/err.txt
    python -c "
import json
try:
  d=json.load(open('gpurun_out/l2fwd/${w}_$pf.json')); k=d['kernels']; print('$w $pf', 'value=%.4g'%d['value'], 'fwd %.3f bwd %.3f step %.3f'%(k['fwd_frac'],k['bwd_frac'],k['step_frac']), d['clocks']['sm_mhz'])
except Exception as e: print('$w ERR', e)
"
  done
done
unset COTTEN_L2_AHEAD
