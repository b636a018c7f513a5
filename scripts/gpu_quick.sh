# quick loop: GPU parity tests + the three bench workloads (+ optional ncu of the d32 kernels)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --workload ml20m --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_ml20m.json 2>> gpurun_out/bench.err
timeout 300 python bench.py --workload beauty --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_beauty.json 2>> gpurun_out/bench.err
if [ "${PROFILE:-0}" = "1" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:d32 -s 2 -c 2 -o gpurun_out/prof_ml20m -f python bench.py --workload ml20m --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>> gpurun_out/bench.err
fi
tail -3 gpurun_out/pytest_gpu.log
for f in bench bench_ml20m bench_beauty; do python -c "
import json; d=json.load(open('gpurun_out/$f.json')); k=d['kernels']; print('$f', 'value=%.4g'%d['value'], 'ms=%.4f'%d['ms_per_step'], 'fwd %.1fus %.3f'%(k['fwd_us'],k['fwd_frac']), 'bwd %.1fus %.3f'%(k['bwd_us'],k['bwd_frac']), 'step %.3f'%k['step_frac'], d['clocks'])" 2>&1 | tail -1; done
tail -3 gpurun_out/bench.err
