# e2e with persistent workers: more threads and the gate
mkdir -p gpurun_out/ep2
one() {
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --no-cpu --no-steady --no-encoder > gpurun_out/ep2/$tag.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ep2/$tag.json')); print('$tag', round(d['e2e']['value']), d['e2e']['repeats_seq_per_s'])"
}
one w4 COTTEN_E2E_THREADS=4
one w8 COTTEN_E2E_THREADS=8
one w8_g8 COTTEN_E2E_THREADS=8 COTTEN_HOST_MAX_CONCURRENT=8
one w3 COTTEN_E2E_THREADS=3
one w4_s4 COTTEN_E2E_THREADS=4 COTTEN_HOST_MAX_SLICES=4
one w4_s16 COTTEN_E2E_THREADS=4 COTTEN_HOST_MAX_SLICES=16
for w in ml20m beauty; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-steady --no-encoder > gpurun_out/ep2/$w.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ep2/$w.json')); print('$w', round(d['e2e']['value']), d['e2e']['repeats_seq_per_s'])"
done
