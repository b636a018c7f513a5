"""Warp-stall samples per CUDA source line (top reasons) from an ncu report.
Usage: python scripts/ncu_stall_lines.py REP KERNEL_REGEX [top]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", "regex:" + kern], capture_output=True, text=True).stdout
hdr, res = None, []
for r in csv.reader(out.splitlines()):
    if "Warp Stall Sampling (All Samples)" in r:
        hdr = r
        iS, iA = r.index("Source"), r.index("Warp Stall Sampling (All Samples)")
        reasons = [(i, h[6:]) for i, h in enumerate(r) if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if hdr and r and r[0].isdigit():
        try:
            a = int(r[iA] or 0)
        except ValueError:
            continue
        if a > 0:
            rs = sorted(((int(r[i] or 0), h) for i, h in reasons), reverse=True)[:3]
            res.append((a, int(r[0]), r[iS].strip()[:80], rs))
tot = sum(x[0] for x in res)
print(f"{kern}: {tot} samples")
for a, ln, src, rs in sorted(res, reverse=True)[:top]:
    print(f"{100 * a / tot:5.1f}% line {ln:4d} {src:80s} {rs}")
