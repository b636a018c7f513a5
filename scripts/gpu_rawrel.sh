# fwd pass-2 raw stage released by the splitter: parity + ML-1M / ML-20M / long4k (3 reps) + trace
mkdir -p gpurun_out/rawrel
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_schedule.py -q -p no:cacheprovider -x > gpurun_out/rawrel/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/rawrel/pytest.log
tail -2 gpurun_out/rawrel/pytest.log
for rep in 1 2 3; do
  for w in ml1m ml20m long4k; do
    timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu --no-steady --no-encoder > gpurun_out/rawrel/${w}_$rep.json 2>>gpurun_out/rawrel/err.txt
    python -c "
import json
d=json.load(open('gpurun_out/rawrel/${w}_$rep.json')); k=d['kernels']; print('$w $rep', 'value=%.4g'%d['value'], 'fwd %.1fus %.3f bwd %.1fus %.3f step %.3f'%(k['fwd_us'],k['fwd_frac'],k['bwd_us'],k['bwd_frac'],k['step_frac']))" 2>&1 | tail -1
  done
done
mkdir -p gpurun_out/rawrel/trace_ml1m
COTTEN_LIB=$PWD/build_variants/lib_trace.so COTTEN_TRACE_DIR=$PWD/gpurun_out/rawrel/trace_ml1m timeout 300 python bench.py --workload ml1m --steps 2 --warmup 3 --no-e2e --no-cpu --no-steady --no-encoder --graph off > /dev/null 2>>gpurun_out/rawrel/err.txt
python scripts/dev/trace_report.py gpurun_out/rawrel/trace_ml1m > gpurun_out/rawrel/trace_ml1m.txt 2>&1; grep -A18 'fwd: slowest' gpurun_out/rawrel/trace_ml1m.txt; grep 'CTA timeline' gpurun_out/rawrel/trace_ml1m.txt
