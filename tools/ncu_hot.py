"""Summarise an ncu --set full report: top SASS instructions by warp-stall samples."""
import csv, subprocess, sys
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]
si = h.index("Warp Stall Sampling (All Samples)"); ie = h.index("Instructions Executed")
data = []
for r in rows[hi + 1:]:
    if len(r) != len(h): continue
    try: data.append((float(r[si] or 0), r[0], r[1], r[ie]))
    except ValueError: pass
tot = sum(d[0] for d in data) or 1
print("total samples", tot)
for d in sorted(data, reverse=True)[:n]:
    print(f"{100*d[0]/tot:5.1f}%  {d[1]}  {d[2][:90]:90s} exec={d[3]}")
