# A/B: store-warp tail waits for smem reads only (default) vs full completion (lib_fullwait);
# per-item timeline of the slowest CTA at ML-1M (lib_trace)
mkdir -p gpurun_out/tail
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_schedule.py -q -p no:cacheprovider -x > gpurun_out/tail/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/tail/pytest.log
tail -2 gpurun_out/tail/pytest.log
for rep in 1 2 3; do
  for v in default fullwait; do
    if [ $v = default ]; then unset COTTEN_LIB; else export COTTEN_LIB=$PWD/build_variants/lib_$v.so; fi
    for w in ml1m ml20m; do
      timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu --no-steady --no-encoder > gpurun_out/tail/${v}_${w}_$rep.json 2>>gpurun_out/tail/err.txt
      python -c "
import json
d=json.load(open('gpurun_out/tail/${v}_${w}_$rep.json')); k=d['kernels']; print('$v $w $rep', 'value=%.4g'%d['value'], 'ms %.4f'%d['ms_per_step'], 'fwd %.1fus %.3f bwd %.1fus %.3f step %.3f'%(k['fwd_us'],k['fwd_frac'],k['bwd_us'],k['bwd_frac'],k['step_frac']))" 2>&1 | tail -1
    done
  done
done
unset COTTEN_LIB
mkdir -p gpurun_out/tail/trace_ml1m
COTTEN_LIB=$PWD/build_variants/lib_trace.so COTTEN_TRACE_DIR=$PWD/gpurun_out/tail/trace_ml1m timeout 300 python bench.py --workload ml1m --steps 2 --warmup 3 --no-e2e --no-cpu --no-steady --no-encoder --graph off > /dev/null 2>>gpurun_out/tail/err.txt
python scripts/dev/trace_report.py gpurun_out/tail/trace_ml1m > gpurun_out/tail/trace_ml1m.txt 2>&1; tail -60 gpurun_out/tail/trace_ml1m.txt
