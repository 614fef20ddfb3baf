"""Summarise an ncu --set full report: top SASS instructions by warp-stall samples.

  python tools/ncu_hot.py <report.ncu-rep> [n_lines] [kernel-regex] [occurrence]

The source page holds one table per profiled launch ("Kernel Name" line, then "Address" header);
kernel-regex / occurrence pick the table (default: the first).
"""
import csv, re, subprocess, sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.abspath(__file__)))
from ncu_page import page  # noqa: E402
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
pat = re.compile(sys.argv[3]) if len(sys.argv) > 3 else None
occ = int(sys.argv[4]) if len(sys.argv) > 4 else 0
out = page(rep, "source", ("--print-source", "sass"))
rows = list(csv.reader(out.splitlines()))
tables, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r[1], None, []]
        tables.append(cur)
    elif r and r[0] == "Address" and cur is not None:
        cur[1] = r
    elif cur is not None and cur[1] is not None and len(r) >= len(cur[1]) - 1:
        cur[2].append(r)
sel = [t for t in tables if pat is None or pat.search(t[0])]
name, h, data = sel[occ]
print(name[:140])
si = h.index("Warp Stall Sampling (All Samples)"); ie = h.index("Instructions Executed")
stalls = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
recs = []
for r in data:
    try:
        recs.append((float(r[si] or 0), r))
    except ValueError:
        pass
tot = sum(x[0] for x in recs) or 1
print("total samples", tot)
agg = {h[i]: sum(float(r[i] or 0) for _, r in recs) for i in stalls}
print("stall mix:", ", ".join(f"{k[6:]} {100 * v / tot:.1f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
for s, r in sorted(recs, key=lambda x: -x[0])[:n]:
    top = sorted(((float(r[i] or 0), h[i][6:]) for i in stalls), reverse=True)[:2]
    print(f"{100 * s / tot:5.1f}%  {r[0]}  {r[1][:80]:80s} exec={r[ie]} [{', '.join(f'{b} {a:.0f}' for a, b in top)}]")
