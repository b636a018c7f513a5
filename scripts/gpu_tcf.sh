# fp32 d_h=64 on tcgen05 (bf16x3): probes, parity, A/B bench vs the register-tiled kernels
mkdir -p gpurun_out/tcf
timeout 60 ./scripts/dev/tmem_ld_probe > gpurun_out/tcf/tmem_ld_probe.txt 2>&1; cat gpurun_out/tcf/tmem_ld_probe.txt
timeout 900 python -m pytest tests/test_gpu_tcf.py -q -p no:cacheprovider -x > gpurun_out/tcf/pytest_tcf.log 2>&1; echo "rc=$?" >> gpurun_out/tcf/pytest_tcf.log
tail -25 gpurun_out/tcf/pytest_tcf.log
for n in 512 4096; do
  w=sw_n${n}_d64_f32
  timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/tcf/$w.json 2>gpurun_out/tcf/$w.err
  python -c "
import json
try:
  d=json.load(open('gpurun_out/tcf/$w.json')); k=d['kernels']; print('$w', 'value=%.4g'%d['value'], 'fwd %.3f bwd %.3f step %.3f'%(k['fwd_frac'],k['bwd_frac'],k['step_frac']), d['clocks']['sm_mhz'])
except Exception as e: print('$w ERR', e)
"
  tail -2 gpurun_out/tcf/$w.err
done
