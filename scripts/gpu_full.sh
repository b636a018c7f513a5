# Full round check: GPU tests, smoke, both bench arms, launch lists + ncu of the tcgen05 kernels.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.csv 2>&1
timeout 600 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 400 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 400 python bench.py --impl reference > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
timeout 300 python bench.py --workload ml20m --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_ml20m.json 2>> gpurun_out/bench.err
timeout 300 python bench.py --workload beauty --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_beauty.json 2>> gpurun_out/bench.err
for w in long4k long16k long4k_d64 long4k_d128; do timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_$w.json 2>> gpurun_out/bench.err; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_ml1m.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-steady --graph off > /dev/null 2>> gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:tc_kernel -c 8 --csv --log-file gpurun_out/launches_ml20m.csv python bench.py --workload ml20m --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>> gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:tc_kernel -s 4 -c 4 --csv --log-file gpurun_out/metrics_ml1m.csv python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --no-steady --graph off > /dev/null 2>> gpurun_out/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_kernel -s 2 -c 2 -o gpurun_out/prof_ml20m -f python bench.py --workload ml20m --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>> gpurun_out/bench.err
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log | tail -2
for f in bench bench_ml20m bench_beauty bench_long4k bench_long16k bench_long4k_d64 bench_long4k_d128; do python -c "
import json; d=json.load(open('gpurun_out/$f.json')); k=d['kernels']; print('$f', 'value=%.4g'%d['value'], 'ms=%.4f'%d['ms_per_step'], 'fwd %.1fus %.3f'%(k['fwd_us'],k['fwd_frac']), 'bwd %.1fus %.3f'%(k['bwd_us'],k['bwd_frac']), 'step %.3f'%k['step_frac'], 'e2e', d.get('e2e',{}).get('value'), 'cpu', d.get('cpu_baseline',{}).get('value'), 'launches', d.get('gpu_launches'), d.get('clocks'))" 2>&1 | tail -1; done
cat gpurun_out/bench_ref.json; tail -3 gpurun_out/bench.err
