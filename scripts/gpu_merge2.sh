mkdir -p gpurun_out/merge
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/merge/pytest_all.log 2>&1; echo "rc=$?" >> gpurun_out/merge/pytest_all.log
tail -8 gpurun_out/merge/pytest_all.log
timeout 600 python bench.py --workload beauty --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/merge/beauty2.json 2>>gpurun_out/merge/err.txt
python -c "
import json
d=json.load(open('gpurun_out/merge/beauty2.json')); k=d['kernels']; print('beauty', 'value=%.4g'%d['value'], 'fwd %.3f bwd %.3f step %.3f'%(k['fwd_frac'],k['bwd_frac'],k['step_frac']), d['run']['kernel_path'], d.get('roofline_max',{}).get('step_frac'))"
