# e2e through the cached host path from W host threads, with the host-call gate
# at its default (4) and disabled (64)
mkdir -p gpurun_out/gate
python -m pytest tests/test_gpu_boundary.py -q -x 2>&1 | tail -2
for G in 4 64; do
for W in 2 4 8 16; do
  COTTEN_HOST_MAX_CONCURRENT=$G COTTEN_E2E_THREADS=$W timeout 600 python bench.py --no-cpu --no-steady --no-encoder --steps 20 --warmup 3 > gpurun_out/gate/g${G}_w$W.json 2>>gpurun_out/gate/err.txt
  python -c "
import json; d=json.load(open('gpurun_out/gate/g${G}_w$W.json')); print('G=$G W=$W', d['value'], d['e2e']['value'], d['e2e'].get('host_threads'))"
done
done
tail -3 gpurun_out/gate/err.txt
