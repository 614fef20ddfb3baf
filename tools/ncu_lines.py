"""Aggregate an ncu --set full report's warp-stall samples by CUDA source line (needs -lineinfo).

  python tools/ncu_lines.py <report.ncu-rep> [n_lines]

Prints the top source lines by stall samples with their dominant stall reasons, so the cost of
one warp role (producer / MMA / expanders / epilogue) can be read off by line range.
"""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr, cur, agg = None, None, None, {}
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        si = hdr.index("Warp Stall Sampling (All Samples)")
        stalls = [i for i, c in enumerate(hdr) if c.startswith("stall_") and "Not Issued" not in c]
        continue
    if hdr is None or len(r) < len(hdr) - 1 or r[0] == "Function Name":
        continue
    if r[0]:   # a source line row (its samples are the sum of its SASS rows)
        try:
            s = float(r[si] or 0)
        except ValueError:
            continue
        key = (fname, int(r[0]))
        st = {hdr[i][6:]: float(r[i] or 0) for i in stalls if r[i] not in ("", "-")}
        e = agg.setdefault(key, [0.0, r[1][:90], {}])
        e[0] += s
        for k, v in st.items():
            e[2][k] = e[2].get(k, 0.0) + v
tot = sum(v[0] for v in agg.values()) or 1.0
print("total samples", tot)
for (f, ln), (s, src, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    top = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{100 * s / tot:5.1f}% {f}:{ln:<5d} {src.strip()[:70]:70s} [{', '.join(f'{k} {100 * v / max(s, 1):.0f}%' for k, v in top)}]")
