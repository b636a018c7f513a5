# e2e (median of 5 repeats) against host threads W, host-call gate 4 vs off
mkdir -p gpurun_out/gate3
for G in 4 64; do
for W in 1 2 4 8 16; do
  tag=g${G}_w$W
  COTTEN_HOST_MAX_CONCURRENT=$G COTTEN_E2E_THREADS=$W timeout 300 python bench.py --no-cpu --no-steady --no-encoder --steps 20 --warmup 3 > gpurun_out/gate3/$tag.json 2>>gpurun_out/gate3/err.txt
  python -c "
import json; d=json.load(open('gpurun_out/gate3/$tag.json')); print('$tag', round(d['e2e']['value']), d['e2e']['repeats_seq_per_s'])"
done
done
tail -3 gpurun_out/gate3/err.txt
