# tail split of the fp32 d_h=32 tcgen05 kernels: full GPU suite + same-box A/B (COTTEN_NO_SPLIT)
mkdir -p gpurun_out/split
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/split/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/split/pytest.log
tail -3 gpurun_out/split/pytest.log
for rep in 1 2; do
  for v in split nosplit; do
    if [ $v = nosplit ]; then export COTTEN_NO_SPLIT=1; else unset COTTEN_NO_SPLIT; fi
    for w in ml1m long16k sw_n8192_d32_f32 sw_n16384_d32_f32 ml20m; do
      timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu --no-steady --no-encoder > gpurun_out/split/${v}_${w}_$rep.json 2>>gpurun_out/split/err.txt
      python -c "
import json
d=json.load(open('gpurun_out/split/${v}_${w}_$rep.json')); k=d['kernels']; print('$v $w $rep', 'value=%.4g'%d['value'], 'fwd %.1fus %.3f bwd %.1fus %.3f step %.3f'%(k['fwd_us'],k['fwd_frac'],k['bwd_us'],k['bwd_frac'],k['step_frac']), d['clocks']['sm_mhz'])" 2>&1 | tail -1
    done
  done
done
unset COTTEN_NO_SPLIT
