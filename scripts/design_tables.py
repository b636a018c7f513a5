"""Regenerate DESIGN.md's "Measured" workload table and config #5 sweep table
from a measurement record (gpurun_out/final as written by
scripts/gpu_round2_final.sh).  Usage: python scripts/design_tables.py [dir]"""
import json
import sys

F = (sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/final").rstrip("/") + "/"


def ld(w):
    return json.load(open(F + ("bench.json" if w == "ml1m" else "bench_%s.json" % w)))


def fmt(v):
    if v >= 1e6:
        return "%.2f M" % (v / 1e6)
    if v >= 1e5:
        return "%.0f k" % (v / 1e3)
    if v >= 1e3:
        return "%.1f k" % (v / 1e3)
    return "%.0f" % v


ROWS = [("ml1m", "ML-1M op (config #2, bench default: 2 layers, B=256)", "tc"),
        ("ml1m_d64", "ML-1M, d_h = 64 reading (H = 1, B=256)", "tcf"),
        ("ml20m", "ML-20M (config #4, B=65536)", "tc"),
        ("beauty", "Beauty (config #3, B=8192, N=50)", "tcf, head pairs merged"),
        ("long4k", "long4k (N=4096, d_h 32, B=1024)", "tc"),
        ("long16k", "long16k (N=16384, d_h 32, B=256)", "tc"),
        ("long4k_d64", "long4k_d64 (d_h 64 fp32, B=512)", "tcf"),
        ("long4k_bf16", "long4k_bf16 (d_h 32 bf16, B=1024)", "tcb paired rows"),
        ("long4k_d64_bf16", "long4k_d64_bf16 (B=512)", "tcb"),
        ("long4k_d128", "long4k_d128 (d_h 128 fp32, B=256)", "tcg"),
        ("long4k_d128_bf16", "long4k_d128_bf16 (B=256)", "tch")]
out = []
for w, name, k in ROWS:
    d = ld(w)
    kk = d["kernels"]
    cap = " *" if d["clocks"].get("reasons") else ""
    val = fmt(d["value"]) + " seq/s"
    if w == "ml1m":
        val = "**" + val + "**"
    out.append("| %s%s | %s | %s | %.3f | %.3f | %.3f | %s seq/s | %s seq/s |" % (
        name, cap, k, val, kk["fwd_frac"], kk["bwd_frac"], kk["step_frac"], fmt(d["e2e"]["value"]),
        fmt(d["cpu_baseline"]["value"])))
e = ld("ml1m")["encoder_step"]
out.append("| encoder training step (config #2 in full) | encoder.cu + tc | %s seq/s (%.2f ms) | — | — | "
           "op %.1f %% of the step | %s seq/s | %s seq/s |" % (
               fmt(e["value"]), e["ms_per_step"], 100 * e["op_kernels"]["share_of_step"],
               fmt(e["e2e"]["value"]), fmt(e["cpu_baseline"]["value"])))
s = open("DESIGN.md").read()
i = s.index("| ML-1M op (config #2, bench default")
j = s.index("\n\n", i)
s = s[:i] + "\n".join(out) + s[j:]
vals = {}
for line in open(F + "sweep_table.md").read().splitlines():
    c = [x.strip() for x in line.strip("|").split("|")]
    if len(c) > 8 and c[0].isdigit():
        vals[(int(c[1]), c[2], int(c[0]))] = c[7]
names = {(32, "f32"): "tc", (64, "f32"): "tcf", (128, "f32"): "tcg", (32, "bf16"): "tcb paired rows",
         (64, "bf16"): "tcb", (128, "bf16"): "tch"}
for (d_, dt), nm in names.items():
    lab = "| %d, %s | %s |" % (d_, "fp32" if dt == "f32" else "bf16", nm)
    k = s.index(lab)
    k2 = s.index("\n", k)
    s = s[:k] + lab + " " + " | ".join(vals[(d_, dt, n)] for n in (512, 1024, 2048, 4096, 8192, 16384)) + " |" + s[k2:]
open("DESIGN.md", "w").write(s)
print("\n".join(out))
