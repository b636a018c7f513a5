# pass-1 slots released before the S epilogue: parity + A/B bench (COTTEN baseline numbers from profiles)
mkdir -p gpurun_out/early
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/early/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/early/pytest.log
tail -3 gpurun_out/early/pytest.log
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/early/bench_ml1m.json 2>gpurun_out/early/bench.err
for w in ml20m sw_n4096_d32_f32 sw_n4096_d64_f32 sw_n4096_d64_bf16 sw_n16384_d32_f32; do
  timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu --no-steady > gpurun_out/early/$w.json 2>>gpurun_out/early/bench.err
done
for f in gpurun_out/early/*.json; do python -c "
import json
try:
  d=json.load(open('$f')); k=d['kernels']; print('$f', 'value=%.4g'%d['value'], 'fwd %.3f bwd %.3f step %.3f'%(k['fwd_frac'],k['bwd_frac'],k['step_frac']), d['clocks']['sm_mhz'], d['clocks']['reasons'])
  s=d.get('steady_state')
  if s: print('   steady', s['value'], s['fwd_frac'], s['bwd_frac'], s['step_frac_of_hbm'])
except Exception as e: print('$f ERR', e)
"; done
