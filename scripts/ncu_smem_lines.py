"""Shared-memory wavefronts per CUDA source line (excessive = bank conflicts) from an ncu report.
Usage: python scripts/ncu_smem_lines.py REP KERNEL_REGEX [top]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg, hdr, cur = {}, None, None
for r in rows:
    if len(r) > 3 and r[0] == "Address" or (len(r) > 3 and r[0] == "Line No"):
        hdr = r
        continue
    if not hdr or len(r) < len(hdr) // 2:
        continue
    if hdr[0] == "Line No":
        cur = (r[0], r[1].strip()[:80])
        continue
if not agg:
    # cuda,sass: sass rows follow their cuda line; fall back to walking both blocks
    pass
iE = iW = None
line = None
res = {}
for r in rows:
    if not r:
        continue
    if "L1 Wavefronts Shared Excessive" in r:
        hdr = r
        iE, iW = r.index("L1 Wavefronts Shared Excessive"), r.index("L1 Wavefronts Shared")
        iS = r.index("Source")
        continue
    if iE is None or len(r) <= iW:
        continue
    if r[0].isdigit():  # a CUDA source line
        line = (int(r[0]), r[iS].strip()[:90])
        try:
            e, w = int(r[iE] or 0), int(r[iW] or 0)
        except ValueError:
            continue
        if w:
            res[line] = (e, w)
tot_e = sum(v[0] for v in res.values())
tot_w = sum(v[1] for v in res.values())
print(f"{kern}: shared wavefronts {tot_w}, excessive {tot_e} ({tot_e / max(tot_w, 1):.1%})")
for (ln, src), (e, w) in sorted(res.items(), key=lambda x: -x[1][0])[:top]:
    print(f"  line {ln:5d} excess {e:11d} of {w:11d}  {src}")
