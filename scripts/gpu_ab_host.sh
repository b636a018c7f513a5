# e2e (host entry points) vs slice size / count: ML-1M default bench, e2e only (2 reps each)
CFGS=("2048 8" "3072 8" "4096 4" "7000 2" "100000 1")
for cfg in "${CFGS[@]}"; do
  set -- $cfg
  for rep in 1 2; do
    COTTEN_HOST_SLICE_KB=$1 COTTEN_HOST_MAX_SLICES=$2 timeout 300 python bench.py --steps 10 --no-cpu --no-steady > gpurun_out/abh_$1_$rep.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/abh_$1_$rep.json')); print('slice $1 KB max $2:', 'e2e %.4g' % d['e2e']['value'])"
  done
done
