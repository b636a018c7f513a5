# tcf backward, one-chunk units: next unit's pass 1 before this unit's pass 2
timeout 600 python -m pytest tests/test_gpu_tcf.py -q -x --timeout 120 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_schedule.py -q --timeout 300 -k "tiny or N1 or beauty or merged" 2>&1 | tail -2
mkdir -p gpurun_out/tcf1
for w in beauty sw_n512_d64_f32; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/tcf1/$w.json 2>gpurun_out/tcf1/$w.err
  python -c "
import json; d=json.load(open('gpurun_out/tcf1/$w.json')); k=d['kernels']; print('$w', round(d['value']), 'fwd %.3f bwd %.3f step %.3f' % (k['fwd_frac'], k['bwd_frac'], k['step_frac']), d['clocks']['sm_mhz'])"
done
