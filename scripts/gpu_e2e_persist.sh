# e2e with persistent host worker threads: W = 1, 2, 4 (median of 7 windows)
mkdir -p gpurun_out/ep
for W in 1 2 4 1; do
  COTTEN_E2E_THREADS=$W timeout 300 python bench.py --no-cpu --no-steady --no-encoder > gpurun_out/ep/w$W.json 2>gpurun_out/ep/err.txt
  python -c "
import json; d=json.load(open('gpurun_out/ep/w$W.json')); print('W=$W', round(d['e2e']['value']), d['e2e']['repeats_seq_per_s'])"
done
tail -2 gpurun_out/ep/err.txt
timeout 120 python scripts/dev/pcie_windows.py | tail -3
