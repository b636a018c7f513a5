# Round-2 measurement record: GPU suite, smoke, default bench + reference arm, every workload line,
# the config #5 sweep, the ncu launch list of the default bench command.
rm -rf gpurun_out/final gpurun_out/sweep
mkdir -p gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/final/gpu.csv 2>&1
timeout 2400 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/final/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final/smoke.log
timeout 900 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/final/bench_ref.json 2>> gpurun_out/final/bench.err
for w in ml1m_d64 ml20m beauty long4k long16k long4k_d64 long4k_d128 long4k_bf16 long4k_d64_bf16 long4k_d128_bf16; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-steady --no-encoder > gpurun_out/final/bench_$w.json 2>> gpurun_out/final/bench.err
done
mkdir -p gpurun_out/sweep
for n in 512 1024 2048 4096 8192 16384; do for d in 32 64 128; do for dt in f32 bf16; do
  w=sw_n${n}_d${d}_${dt}
  timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/sweep/$w.json 2>gpurun_out/sweep/$w.err
done; done; done
python scripts/sweep_table.py gpurun_out/sweep > gpurun_out/final/sweep_table.md
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/final/launches_default.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-steady --no-encoder > /dev/null 2>> gpurun_out/final/bench.err
tail -3 gpurun_out/final/pytest_gpu.log; tail -1 gpurun_out/final/smoke.log
python - <<'PY'
import json, glob
for f in ['gpurun_out/final/bench.json'] + sorted(glob.glob('gpurun_out/final/bench_*.json')):
    try:
        d = json.load(open(f)); k = d.get('kernels', {})
        print(f.split('/')[-1], 'value=%.4g' % d['value'], 'fwd %.3f bwd %.3f step %.3f' % (k.get('fwd_frac', 0), k.get('bwd_frac', 0), k.get('step_frac', 0)),
              'e2e', (d.get('e2e') or {}).get('value'), 'cpu', (d.get('cpu_baseline') or {}).get('value'), d.get('clocks', {}).get('sm_mhz'), d.get('clocks', {}).get('reasons'))
    except Exception as e:
        print(f, 'ERR', e)
PY
