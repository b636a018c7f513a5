# tcg backward with direct global stores and early slot release: parity, bench, trace
timeout 600 python -m pytest tests/test_gpu_tcg.py -q -x --timeout 120 2>&1 | tail -2
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundary.py -q --timeout 120 -k "128" 2>&1 | tail -1
mkdir -p gpurun_out/tcg5
for w in long4k_d128 sw_n512_d128_f32 sw_n2048_d128_f32 sw_n16384_d128_f32; do
  timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/tcg5/$w.json 2>gpurun_out/tcg5/$w.err
  python -c "
import json; d=json.load(open('gpurun_out/tcg5/$w.json')); k=d['kernels']; print('$w', round(d['value']), 'fwd %.3f bwd %.3f step %.3f' % (k['fwd_frac'], k['bwd_frac'], k['step_frac']), d['clocks']['sm_mhz'])"
done
mkdir -p gpurun_out/tgt2
COTTEN_LIB=build_variants/lib_tcgtrace.so COTTEN_TRACE_DIR=gpurun_out/tgt2 timeout 300 python bench.py --workload sw_n2048_d128_f32 --steps 1 --warmup 1 --no-e2e --no-cpu --graph off > /dev/null 2>&1
python scripts/dev/tcb_trace_report.py gpurun_out/tgt2 | head -14
