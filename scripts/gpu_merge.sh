# head-merged fp32 d_h=32 (Beauty) on tcgen05: parity + bench vs the FP32-pipe d32 kernels
mkdir -p gpurun_out/merge
timeout 900 python -m pytest tests/test_gpu_tcf.py -q -p no:cacheprovider -x > gpurun_out/merge/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/merge/pytest.log
tail -15 gpurun_out/merge/pytest.log
timeout 600 python bench.py --workload beauty --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/merge/beauty.json 2>gpurun_out/merge/err.txt
timeout 600 python bench.py --workload beauty --steps 10 --warmup 3 --no-e2e --no-cpu --path fp32pipe > gpurun_out/merge/beauty_fp32pipe.json 2>>gpurun_out/merge/err.txt
for f in beauty beauty_fp32pipe; do python -c "
import json
try:
  d=json.load(open('gpurun_out/merge/$f.json')); k=d['kernels']; print('$f', 'value=%.4g'%d['value'], 'fwd %.3f bwd %.3f step %.3f'%(k['fwd_frac'],k['bwd_frac'],k['step_frac']), d['run']['kernel_path'], d['clocks']['sm_mhz'])
except Exception as e: print('$f ERR', e)
"; done
tail -3 gpurun_out/merge/err.txt
