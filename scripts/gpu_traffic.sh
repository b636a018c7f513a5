# DRAM bytes per launch of the tcgen05 kernels per workload (profiles/traffic.json)
mkdir -p gpurun_out/traffic
for w in ml1m ml20m beauty long4k long4k_d64 long4k_bf16 long4k_d64_bf16 ml1m_d64; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"tc_kernel|tcf_kernel|tcb_kernel" -c 6 --csv --log-file gpurun_out/traffic/$w.csv python bench.py --workload $w --steps 1 --warmup 1 --no-e2e --no-cpu --no-steady --no-encoder --graph off > /dev/null 2>> gpurun_out/traffic/err.txt
done
ls -la gpurun_out/traffic
