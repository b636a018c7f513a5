# d_h=128 register-tiled kernels at 512 threads per CTA vs 256 (lib_rt256): parity + bench
mkdir -p gpurun_out/rt512
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_schedule.py -q -p no:cacheprovider -k "128 or head_dims or bf16" > gpurun_out/rt512/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/rt512/pytest.log
tail -3 gpurun_out/rt512/pytest.log
for rep in 1 2; do
  for v in rt512 rt256; do
    if [ $v = rt256 ]; then export COTTEN_LIB=$PWD/build_variants/lib_rt256.so; else unset COTTEN_LIB; fi
    for w in long4k_d128 long4k_d128_bf16 sw_n16384_d128_f32; do
      timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/rt512/${v}_${w}_$rep.json 2>>gpurun_out/rt512/err.txt
      python -c "
import json
d=json.load(open('gpurun_out/rt512/${v}_${w}_$rep.json')); k=d['kernels']; print('$v $w $rep', 'value=%.4g'%d['value'], 'fwd %.3f bwd %.3f step %.3f'%(k['fwd_frac'],k['bwd_frac'],k['step_frac']), d['roofline_max']['step_frac'])" 2>&1 | tail -1
    done
  done
done
unset COTTEN_LIB
