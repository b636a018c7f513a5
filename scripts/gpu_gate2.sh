# W=8 e2e diagnosis: serialised gate, more hardware queues, one slice per call
mkdir -p gpurun_out/gate2
nproc; nvidia-smi topo -m | head -3
one() {  # tag, env...
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --no-cpu --no-steady --no-encoder --steps 20 --warmup 3 > gpurun_out/gate2/$tag.json 2>>gpurun_out/gate2/err.txt
  python -c "
import json; d=json.load(open('gpurun_out/gate2/$tag.json')); print('$tag', round(d['e2e']['value']))"
}
one w1 COTTEN_E2E_THREADS=1
one w2 COTTEN_E2E_THREADS=2
one w8 COTTEN_E2E_THREADS=8
one w8_g1 COTTEN_E2E_THREADS=8 COTTEN_HOST_MAX_CONCURRENT=1
one w8_g2 COTTEN_E2E_THREADS=8 COTTEN_HOST_MAX_CONCURRENT=2
one w8_conn32 COTTEN_E2E_THREADS=8 CUDA_DEVICE_MAX_CONNECTIONS=32
one w8_s1 COTTEN_E2E_THREADS=8 COTTEN_HOST_MAX_SLICES=1
one w4_s1 COTTEN_E2E_THREADS=4 COTTEN_HOST_MAX_SLICES=1
one w2_again COTTEN_E2E_THREADS=2
tail -3 gpurun_out/gate2/err.txt
