# the backward's saved-S operand written by the mask warp (default) vs by the splitter (lib_prev): tests + A/B
mkdir -p gpurun_out/maskS
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/maskS/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/maskS/pytest.log
tail -3 gpurun_out/maskS/pytest.log
for rep in 1 2; do
  for v in new prev; do
    if [ $v = prev ]; then export COTTEN_LIB=$PWD/build_variants/lib_prev.so; else unset COTTEN_LIB; fi
    for w in ml1m ml20m beauty ml1m_d64 long4k_d64_bf16 long4k_bf16; do
      timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu --no-steady --no-encoder > gpurun_out/maskS/${v}_${w}_$rep.json 2>>gpurun_out/maskS/err.txt
      python -c "
import json
d=json.load(open('gpurun_out/maskS/${v}_${w}_$rep.json')); k=d['kernels']; print('$v $w $rep', 'value=%.4g'%d['value'], 'fwd %.3f bwd %.3f step %.3f'%(k['fwd_frac'],k['bwd_frac'],k['step_frac']), d['clocks']['sm_mhz'])" 2>&1 | tail -1
    done
  done
done
unset COTTEN_LIB
