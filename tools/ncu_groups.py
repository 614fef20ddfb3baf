"""Instruction mix of one kernel of an ncu report: executed warp-instructions grouped by runs of
SASS lines with equal execution counts (basic blocks), largest first.
  python tools/ncu_groups.py <report.ncu-rep> <units> [n]   (units: divide counts by this, e.g. warp-elements)"""
import csv, subprocess, sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.abspath(__file__)))
from ncu_page import page  # noqa: E402
rep, units = sys.argv[1], float(sys.argv[2])
n = int(sys.argv[3]) if len(sys.argv) > 3 else 14
out = page(rep, "source", ("--print-source", "sass"))
h, data = None, []
for r in csv.reader(out.splitlines()):
    if r and r[0] == "Address":
        h = r
        continue
    if h and len(r) >= len(h) - 1:
        data.append(r)
ie = h.index("Instructions Executed")
tot, groups = 0.0, []
for r in data:
    try:
        e = float(r[ie] or 0)
    except ValueError:
        continue
    tot += e
    if groups and groups[-1][0] == e:
        groups[-1][1] += 1
        groups[-1][2].append(r[1])
    else:
        groups.append([e, 1, [r[1]]])
print(f"total {tot:.0f} warp-instructions = {tot / units:.1f} per unit")
for e, k, ss in sorted(groups, key=lambda g: -g[0] * g[1])[:n]:
    print(f"{e:10.0f} x {k:4d} = {e * k / units:6.1f}/unit   {ss[0][:48]} ... {ss[-1][:40]}")
