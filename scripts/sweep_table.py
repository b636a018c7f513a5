"""Table of the config #5 sweep lines (bench.py --workload sw_n*_d*_*)."""
import glob
import json
import os
import sys

rows = []
for f in sorted(glob.glob(os.path.join(sys.argv[1], "sw_*.json"))):
    try:
        d = json.load(open(f))
    except Exception:
        continue
    c = d["config"]
    k = d.get("kernels", {})
    rm = d.get("roofline_max", {})
    rows.append((c["seq_len"], c["head_dim"], c["dtype"], c["global_batch"], d["value"],
                 k.get("fwd_frac"), k.get("bwd_frac"), k.get("step_frac"), rm.get("step_frac"),
                 d["run"]["kernel_path"], d["clocks"]["sm_mhz"], ",".join(d["clocks"]["reasons"])))
rows.sort()
print("| N | d_h | dtype | B | seq/s | fwd frac | bwd frac | step frac (HBM) | step frac of max(compute, HBM) (compute = the pipe used) | kernels | SM MHz | throttle |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|")
f = lambda x: "-" if x is None else f"{x:.3f}"  # noqa: E731
for r in rows:
    print(f"| {r[0]} | {r[1]} | {r[2]} | {r[3]} | {r[4]:.4g} | {f(r[5])} | {f(r[6])} | {f(r[7])} | "
          f"{f(r[8])} | {r[9]} | {r[10]:.0f} | {r[11]} |")
