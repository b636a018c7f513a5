"""Per-source-line warp-stall samples (with the top stall reasons) from
`ncu -i REP --page source --csv --print-source cuda,sass [--kernel-name regex:K] > F`.
Usage: python scripts/ncu_lines.py F [top] [first_line last_line]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
lo, hi = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (0, 1 << 30)
fname, res, hdr = None, [], None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        reasons = [(i, h[6:]) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if hdr and r[0]:
        try:
            n = int(r[4])
        except (IndexError, ValueError):
            continue
        ln = int(r[0])
        if fname == "kernels_tc.cuh" and not (lo <= ln <= hi):
            continue
        rs = sorted(((int(r[i]) if r[i].isdigit() else 0, name) for i, name in reasons), reverse=True)[:3]
        res.append((n, fname, ln, r[1][:70], rs))
tot = sum(x[0] for x in res)
print("total stall samples", tot)
for s, f, ln, src, rs in sorted(res, reverse=True)[:top]:
    why = " ".join(f"{nm}:{100 * v / max(s, 1):.0f}%" for v, nm in rs if v)
    print(f"{s:7d} {100 * s / tot:5.1f}%  {f}:{ln:<5} {src:70s} {why}")
