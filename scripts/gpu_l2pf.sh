# A/B of the producers' L2 prefetch distance (COTTEN_L2_AHEAD) on the tcgen05 kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tcb.py tests/test_gpu_schedule.py tests/test_gpu_parity.py -q -p no:cacheprovider -x > gpurun_out/pytest_pf.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pf.log
tail -2 gpurun_out/pytest_pf.log
for w in ml1m ml20m long4k long4k_d64_bf16; do
  for a in 0 4 8; do
    COTTEN_L2_AHEAD=$a timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu --no-steady --no-encoder > gpurun_out/pf_${w}_$a.json 2>/dev/null
    python -c "
import json
d=json.load(open('gpurun_out/pf_${w}_$a.json')); k=d['kernels']; print('$w ahead=$a', 'value=%.4g'%d['value'], 'fwd %.3f bwd %.3f step %.3f'%(k['fwd_frac'],k['bwd_frac'],k['step_frac']), d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1
  done
done
