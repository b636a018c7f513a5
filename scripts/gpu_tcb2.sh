# tcb (bf16 d_h 64): per-unit S / G epilogue on all 128 epiloguer threads
timeout 600 python -m pytest tests/test_gpu_tcb.py -q -x --timeout 120 2>&1 | tail -2
mkdir -p gpurun_out/tcb2
for w in sw_n512_d64_bf16 sw_n4096_d64_bf16 long4k_d64_bf16; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu --no-steady --no-encoder > gpurun_out/tcb2/$w.json 2>gpurun_out/tcb2/$w.err
  python -c "
import json; d=json.load(open('gpurun_out/tcb2/$w.json')); k=d['kernels']; print('$w', round(d['value']), 'fwd %.3f bwd %.3f step %.3f' % (k['fwd_frac'], k['bwd_frac'], k['step_frac']), d['clocks']['sm_mhz'])"
done
