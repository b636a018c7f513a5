# e2e with persistent workers: slice size against thread count
mkdir -p gpurun_out/es
one() {
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --no-cpu --no-steady --no-encoder > gpurun_out/es/$tag.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/es/$tag.json')); print('$tag', round(d['e2e']['value']), d['e2e']['repeats_seq_per_s'])"
}
one w8 COTTEN_E2E_THREADS=8
one w8_s512 COTTEN_E2E_THREADS=8 COTTEN_HOST_SLICE_KB=512
one w8_s1024 COTTEN_E2E_THREADS=8 COTTEN_HOST_SLICE_KB=1024
one w4_s1024 COTTEN_E2E_THREADS=4 COTTEN_HOST_SLICE_KB=1024
one w4_s512 COTTEN_E2E_THREADS=4 COTTEN_HOST_SLICE_KB=512
one w2_s512 COTTEN_E2E_THREADS=2 COTTEN_HOST_SLICE_KB=512
