# e2e (median of 5 repeats) against host threads W: host_wait spin vs auto
mkdir -p gpurun_out/hostsync
cat /sys/fs/cgroup/cpu.max 2>/dev/null; nproc
python -m pytest tests/test_gpu_boundary.py -q -x 2>&1 | tail -1
for M in auto spin block; do
for W in 1 2 4 8 16; do
  tag=${M}_w$W
  COTTEN_HOST_SYNC=$M COTTEN_E2E_THREADS=$W timeout 300 python bench.py --no-cpu --no-steady --no-encoder --steps 20 --warmup 3 > gpurun_out/hostsync/$tag.json 2>>gpurun_out/hostsync/err.txt
  python -c "
import json; d=json.load(open('gpurun_out/hostsync/$tag.json')); print('$tag', round(d['e2e']['value']), d['e2e']['repeats_seq_per_s'])"
done
done
tail -3 gpurun_out/hostsync/err.txt
