# A/B of build_variants/*.so on the register-tiled kernels: long4k_d64 / long4k_d128 / long4k_bf16 (median of 3)
for lib in build_variants/lib_*.so; do
  n=$(basename $lib .so)
  for w in long4k_d64 long4k_d128 long4k_bf16; do
    for rep in 1 2 3; do
      COTTEN_LIB=$PWD/$lib timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/abrt_${n}_${w}_$rep.json 2>/dev/null
    done
    python - <<PY
import json, statistics
ks = [json.load(open(f"gpurun_out/abrt_${n}_${w}_{r}.json"))["kernels"] for r in (1, 2, 3)]
m = lambda key: statistics.median(k[key] for k in ks)
print("${n} ${w}", "fwd %.1fus %.3f" % (m("fwd_us"), m("fwd_frac")), "bwd %.1fus %.3f" % (m("bwd_us"), m("bwd_frac")), "step %.3f" % m("step_frac"))
PY
  done
  COTTEN_LIB=$PWD/$lib timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "head_dim or bf16" -p no:cacheprovider 2>&1 | tail -1
done
