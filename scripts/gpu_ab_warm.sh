# Same-box A/B: L2 warm-up before the programmatic dependency (default) vs none (lib_nowarm)
mkdir -p gpurun_out/abwarm
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_schedule.py tests/test_encoder_gpu.py -q -p no:cacheprovider -x > gpurun_out/abwarm/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/abwarm/pytest.log
tail -2 gpurun_out/abwarm/pytest.log
for rep in 1 2 3; do
  for v in nowarm default; do
    if [ $v = default ]; then unset COTTEN_LIB; else export COTTEN_LIB=$PWD/build_variants/lib_$v.so; fi
    for w in ml1m ml20m; do
      timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu --no-steady --no-encoder > gpurun_out/abwarm/${v}_${w}_$rep.json 2>>gpurun_out/abwarm/err.txt
      python -c "
import json
d=json.load(open('gpurun_out/abwarm/${v}_${w}_$rep.json')); k=d['kernels']; print('$v $w $rep', 'value=%.4g'%d['value'], 'ms %.4f'%d['ms_per_step'], 'fwd %.1fus %.3f bwd %.1fus %.3f step %.3f'%(k['fwd_us'],k['fwd_frac'],k['bwd_us'],k['bwd_frac'],k['step_frac']), d['clocks']['sm_mhz'])" 2>&1 | tail -1
    done
  done
done
unset COTTEN_LIB
