# tcg (two-slot ring): L2 prefetch distance A/B for both kernels
mkdir -p gpurun_out/tcg_l2
for a in 0 2 4 8; do
for w in long4k_d128 sw_n512_d128_f32; do
  COTTEN_L2_AHEAD=$a timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/tcg_l2/${w}_a$a.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/tcg_l2/${w}_a$a.json')); k=d['kernels']; print('$w a=$a', round(d['value']), 'fwd %.3f bwd %.3f step %.3f' % (k['fwd_frac'], k['bwd_frac'], k['step_frac']), d['clocks']['sm_mhz'])"
done
done
