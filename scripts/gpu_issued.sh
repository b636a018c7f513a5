# first-unit loads ahead of the bulk TMA (tc), L2 prefetch of the next unit's S (tcb/tcf bwd)
mkdir -p gpurun_out/issued
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/issued/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/issued/pytest.log
tail -3 gpurun_out/issued/pytest.log
for rep in 1 2; do
  for w in ml1m ml20m beauty long4k_d64_bf16 sw_n4096_d64_f32 long4k_bf16; do
    timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu --no-steady --no-encoder > gpurun_out/issued/${w}_$rep.json 2>>gpurun_out/issued/err.txt
    python -c "
import json
d=json.load(open('gpurun_out/issued/${w}_$rep.json')); k=d['kernels']; print('$w $rep', 'value=%.4g'%d['value'], 'fwd %.1fus %.3f bwd %.1fus %.3f step %.3f'%(k['fwd_us'],k['fwd_frac'],k['bwd_us'],k['bwd_frac'],k['step_frac']), d['clocks']['sm_mhz'])" 2>&1 | tail -1
  done
done
mkdir -p gpurun_out/issued/trace_ml1m
COTTEN_LIB=$PWD/build_variants/lib_trace.so COTTEN_TRACE_DIR=$PWD/gpurun_out/issued/trace_ml1m timeout 300 python bench.py --workload ml1m --steps 2 --warmup 3 --no-e2e --no-cpu --no-steady --no-encoder --graph off > /dev/null 2>>gpurun_out/issued/err.txt
python scripts/dev/trace_report.py gpurun_out/issued/trace_ml1m > gpurun_out/issued/trace_ml1m.txt 2>&1; grep 'CTA timeline' gpurun_out/issued/trace_ml1m.txt
