# bf16 d_h = 128 on tcgen05 (kernels_tch.cuh) against the FP32-pipe partner
mkdir -p gpurun_out/tch
for w in long4k_d128_bf16 sw_n512_d128_bf16 sw_n2048_d128_bf16 sw_n16384_d128_bf16; do
  timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/tch/$w.json 2>gpurun_out/tch/$w.err
  COTTEN_NO_TCH=1 timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/tch/${w}_rt.json 2>>gpurun_out/tch/$w.err
  python - <<PY
import json
for tag in ("$w", "${w}_rt"):
    d = json.load(open("gpurun_out/tch/%s.json" % tag))
    k = d["kernels"]
    print(tag, round(d["value"]), "fwd %.3f bwd %.3f step %.3f" % (k["fwd_frac"], k["bwd_frac"], k["step_frac"]), d.get("kernel_path", d["config"].get("kernels", "")))
PY
done
tail -3 gpurun_out/tch/*.err | head -20
# launch list + one full ncu capture of each tch kernel at long4k_d128_bf16
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/tch/launches.csv python bench.py --workload long4k_d128_bf16 --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cos_.*_tch -c 2 -o gpurun_out/tch/tch_full python bench.py --workload long4k_d128_bf16 --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1
ls -la gpurun_out/tch/
