mkdir -p gpurun_out/trace_ml20m gpurun_out/trace_ml1m
COTTEN_LIB=$PWD/build_variants/lib_trace.so COTTEN_TRACE_DIR=$PWD/gpurun_out/trace_ml20m timeout 300 python bench.py --workload ml20m --steps 2 --warmup 3 --no-e2e --no-cpu --graph off > /dev/null 2>&1
COTTEN_LIB=$PWD/build_variants/lib_trace.so COTTEN_TRACE_DIR=$PWD/gpurun_out/trace_ml1m timeout 300 python bench.py --workload ml1m --steps 2 --warmup 3 --no-e2e --no-cpu --no-steady --graph off > /dev/null 2>&1
echo ML20M; python scripts/dev/trace_report.py gpurun_out/trace_ml20m
echo ML1M; python scripts/dev/trace_report.py gpurun_out/trace_ml1m
