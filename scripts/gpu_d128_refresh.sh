# d_h = 128 after the tcg forward change: DRAM bytes per launch (traffic.json) and the sweep / bench lines
mkdir -p gpurun_out/traffic gpurun_out/sweep gpurun_out/d128
for w in long4k_d128 long4k_d128_bf16; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"tch_kernel|tcg_kernel" -c 6 --csv --log-file gpurun_out/traffic/$w.csv python bench.py --workload $w --steps 1 --warmup 1 --no-e2e --no-cpu --no-steady --no-encoder --graph off > /dev/null 2>> gpurun_out/traffic/err.txt
done
for n in 512 1024 2048 4096 8192 16384; do
  w=sw_n${n}_d128_f32
  timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/sweep/$w.json 2>gpurun_out/sweep/$w.err
done
timeout 600 python bench.py --workload long4k_d128 --steps 10 --warmup 3 --no-steady --no-encoder > gpurun_out/d128/bench_long4k_d128.json 2>gpurun_out/d128/err.txt
python -c "
import json; d=json.load(open('gpurun_out/d128/bench_long4k_d128.json')); k=d['kernels']; print('long4k_d128', d['value'], k, d['e2e']['value'], d['cpu_baseline']['value'], d['clocks'])"
ls gpurun_out/traffic
