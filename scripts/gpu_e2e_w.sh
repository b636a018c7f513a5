# e2e host path: threads W, host-call gate G, slices S (median of 7 windows each)
mkdir -p gpurun_out/ew
one() {
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --no-cpu --no-steady --no-encoder > gpurun_out/ew/$tag.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ew/$tag.json')); print('$tag', round(d['e2e']['value']), d['e2e']['repeats_seq_per_s'])"
}
one w1 COTTEN_E2E_THREADS=1
one w2 COTTEN_E2E_THREADS=2
one w2_g1 COTTEN_E2E_THREADS=2 COTTEN_HOST_MAX_CONCURRENT=1
one w1_s4 COTTEN_E2E_THREADS=1 COTTEN_HOST_MAX_SLICES=4
one w1_s16 COTTEN_E2E_THREADS=1 COTTEN_HOST_MAX_SLICES=16
one w2_s4 COTTEN_E2E_THREADS=2 COTTEN_HOST_MAX_SLICES=4
one w4 COTTEN_E2E_THREADS=4
one w1_again COTTEN_E2E_THREADS=1
