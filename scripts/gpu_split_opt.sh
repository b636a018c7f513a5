# tcf / tcb splitter changes: parity + bench
mkdir -p gpurun_out/splitopt
timeout 900 python -m pytest tests/test_gpu_tcf.py tests/test_gpu_tcb.py -q -p no:cacheprovider -x > gpurun_out/splitopt/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/splitopt/pytest.log
tail -4 gpurun_out/splitopt/pytest.log
for w in sw_n512_d64_f32 sw_n4096_d64_f32 sw_n16384_d64_f32 sw_n4096_d64_bf16 sw_n4096_d32_bf16 sw_n512_d32_bf16; do
  timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/splitopt/$w.json 2>gpurun_out/splitopt/$w.err
  python -c "
import json
try:
  d=json.load(open('gpurun_out/splitopt/$w.json')); k=d['kernels']; print('$w', 'value=%.4g'%d['value'], 'fwd %.3f bwd %.3f step %.3f'%(k['fwd_frac'],k['bwd_frac'],k['step_frac']), d['clocks']['sm_mhz'], d['clocks']['reasons'])
except Exception as e: print('$w ERR', e)
"
done
