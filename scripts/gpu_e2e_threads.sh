# e2e through the cached host path from W host threads
mkdir -p gpurun_out/e2e
for W in 1 2 4 8; do
  COTTEN_E2E_THREADS=$W timeout 600 python bench.py --no-cpu --no-steady --no-encoder --steps 20 --warmup 3 > gpurun_out/e2e/ml1m_w$W.json 2>>gpurun_out/e2e/err.txt
  python -c "
import json; d=json.load(open('gpurun_out/e2e/ml1m_w$W.json')); print('W=$W', d['value'], d['e2e']['value'], d['e2e'].get('host_threads'))"
done
tail -3 gpurun_out/e2e/err.txt
bash scripts/gpu_traffic.sh
python scripts/traffic_json.py gpurun_out/traffic > gpurun_out/traffic/traffic.json; cat gpurun_out/traffic/traffic.json
