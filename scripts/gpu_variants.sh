# A/B of kernel build variants: error table + ML-20M / ML-1M bench per variant library.
mkdir -p gpurun_out
for lib in build_variants/*.so; do
  n=$(basename $lib .so)
  echo "== $n"
  COTTEN_LIB=$PWD/$lib timeout 300 python scripts/dev/err_table.py 2>/dev/null | grep -E "N=  200|N= 2048|N=  513"
  for w in ml20m ml1m; do
    COTTEN_LIB=$PWD/$lib timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/v_${n}_$w.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/v_${n}_$w.json')); k=d['kernels']; print('  $w', 'fwd %.1fus %.3f'%(k['fwd_us'],k['fwd_frac']), 'bwd %.1fus %.3f'%(k['bwd_us'],k['bwd_frac']), 'step %.3f'%k['step_frac'])"
  done
done
