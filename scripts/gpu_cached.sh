# device-resident host cache: boundary tests + default bench (e2e through the cached pair)
mkdir -p gpurun_out/cached
timeout 900 python -m pytest tests/test_gpu_boundary.py tests/test_capi_cpu.py -q -p no:cacheprovider > gpurun_out/cached/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/cached/pytest.log
tail -3 gpurun_out/cached/pytest.log
timeout 900 python bench.py --no-cpu > gpurun_out/cached/bench.json 2> gpurun_out/cached/bench.err
for w in ml20m beauty long4k; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-steady --no-encoder --no-cpu > gpurun_out/cached/bench_$w.json 2>> gpurun_out/cached/bench.err
done
python - <<'PY'
import json, glob
for f in ['gpurun_out/cached/bench.json'] + sorted(glob.glob('gpurun_out/cached/bench_*.json')):
    try:
        d = json.load(open(f)); k = d.get('kernels', {})
        print(f.split('/')[-1], 'value=%.4g' % d['value'], 'step %.3f' % k.get('step_frac', 0), 'e2e', d.get('e2e'))
    except Exception as e:
        print(f, 'ERR', e)
PY
tail -3 gpurun_out/cached/bench.err
