# Same-box A/B of the start-up gate and the early raw release (tc kernels), 3 reps, + start-up trace
mkdir -p gpurun_out/abstart
mkdir -p gpurun_out/abstart/trace_ml1m
COTTEN_LIB=$PWD/build_variants/lib_trace.so COTTEN_TRACE_DIR=$PWD/gpurun_out/abstart/trace_ml1m timeout 300 python bench.py --workload ml1m --steps 2 --warmup 3 --no-e2e --no-cpu --no-steady --no-encoder --graph off > /dev/null 2>>gpurun_out/abstart/err.txt
python scripts/dev/trace_report.py gpurun_out/abstart/trace_ml1m > gpurun_out/abstart/trace_ml1m.txt 2>&1; grep -E 'start-up|CTA timeline' gpurun_out/abstart/trace_ml1m.txt
for rep in 1 2 3; do
  for v in base gate default; do
    if [ $v = default ]; then unset COTTEN_LIB; else export COTTEN_LIB=$PWD/build_variants/lib_$v.so; fi
    for w in ml1m ml20m; do
      timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu --no-steady --no-encoder > gpurun_out/abstart/${v}_${w}_$rep.json 2>>gpurun_out/abstart/err.txt
      python -c "
import json
d=json.load(open('gpurun_out/abstart/${v}_${w}_$rep.json')); k=d['kernels']; print('$v $w $rep', 'value=%.4g'%d['value'], 'fwd %.1fus %.3f bwd %.1fus %.3f step %.3f'%(k['fwd_us'],k['fwd_frac'],k['bwd_us'],k['bwd_frac'],k['step_frac']), d['clocks']['sm_mhz'])" 2>&1 | tail -1
    done
  done
done
unset COTTEN_LIB
