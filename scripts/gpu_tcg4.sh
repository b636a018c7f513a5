# tcg backward: slot-1 items drained by epiloguer warps 2-3
timeout 600 python -m pytest tests/test_gpu_tcg.py -q -x --timeout 120 2>&1 | tail -2
mkdir -p gpurun_out/tcg4
for w in long4k_d128 sw_n512_d128_f32 sw_n2048_d128_f32 sw_n16384_d128_f32; do
  timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/tcg4/$w.json 2>gpurun_out/tcg4/$w.err
  python -c "
import json; d=json.load(open('gpurun_out/tcg4/$w.json')); k=d['kernels']; print('$w', round(d['value']), 'fwd %.3f bwd %.3f step %.3f' % (k['fwd_frac'], k['bwd_frac'], k['step_frac']), d['clocks']['sm_mhz'])"
done
