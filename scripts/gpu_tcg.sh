# fp32 d_h = 128 on tcgen05 (kernels_tcg.cuh): parity + the fp32 d128 points against the FP32-pipe partner
timeout 500 python -m pytest tests/test_gpu_tcg.py -q --timeout 120 2>&1 | tail -3
mkdir -p gpurun_out/tcg
for w in long4k_d128 sw_n512_d128_f32 sw_n2048_d128_f32 sw_n16384_d128_f32; do
  for v in tcg rt; do
    if [ $v = rt ]; then export COTTEN_NO_TCG=1; else unset COTTEN_NO_TCG; fi
    timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/tcg/${w}_$v.json 2>gpurun_out/tcg/${w}_$v.err
    python -c "
import json; d=json.load(open('gpurun_out/tcg/${w}_$v.json')); k=d['kernels']; print('$w $v', round(d['value']), 'fwd %.3f bwd %.3f step %.3f' % (k['fwd_frac'], k['bwd_frac'], k['step_frac']), d['clocks']['sm_mhz'])"
  done
done
unset COTTEN_NO_TCG
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/tcg/launches.csv python bench.py --workload long4k_d128 --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cos_.*_tcg -c 2 -o gpurun_out/tcg/tcg_full python bench.py --workload long4k_d128 --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1
ls gpurun_out/tcg | head -30
