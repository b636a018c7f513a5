# e2e, persistent workers, gate default 8: W = 8, 16, 4
mkdir -p gpurun_out/ep3
for W in 8 16 4 8; do
  COTTEN_E2E_THREADS=$W timeout 300 python bench.py --no-cpu --no-steady --no-encoder > gpurun_out/ep3/w$W.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ep3/w$W.json')); print('W=$W', round(d['e2e']['value']), d['e2e']['repeats_seq_per_s'])"
done
timeout 300 python -m pytest tests/test_gpu_boundary.py -q 2>&1 | tail -1
