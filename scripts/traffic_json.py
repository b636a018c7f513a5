"""profiles/traffic.json from ncu launch lists (gpurun_out/traffic/<workload>.csv):
dram__bytes_read.sum + dram__bytes_write.sum per launch, averaged per kernel kind."""
import collections
import csv
import glob
import json
import os
import sys

src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/traffic"
out = {"_source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (per launch, averaged; "
                  "ncu replays each kernel with flushed caches, so small launches' outputs that stay "
                  "in the 126 MB L2 under ncu still count when written back) of the tcgen05 kernels "
                  "per bench workload: scripts/gpu_traffic.sh, " + src}
for f in sorted(glob.glob(os.path.join(src, "*.csv"))):
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    if not rows:
        continue
    hdr = rows[0]
    ki, mi, vi, ii, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID",
                                                  "Metric Unit"))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    per = collections.defaultdict(dict)
    for r in rows[1:]:
        per[(r[ii], r[ki])][r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
    agg = collections.defaultdict(list)
    for (_, k), m in per.items():
        kind = "bwd" if "bwd" in k else "fwd"
        agg[kind].append(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0))
    out[os.path.basename(f)[:-4]] = {k: int(sum(v) / len(v)) for k, v in agg.items()}
print(json.dumps(out, indent=2))
