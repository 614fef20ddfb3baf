"""Summarise this round's ncu evidence into profiles/ (run here, on the CPU box).

  python tools/ncu_summarize.py <round> <launches.csv> <name=report.ncu-rep>...

Writes profiles/<round>_ncu_summary.md (per-report key metrics with units, and the kernel share
of one step from the cold-cache launch list) and profiles/ncu_traffic.json (DRAM bytes per
launch of each profiled kernel, read by bench.py for roofline.traffic).
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.abspath(__file__)))
from ncu_page import page  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__cycles_elapsed.avg.per_second"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9, "second": 1.0}


def raw(rep):
    """Metrics of the report's first kernel; with several kernels in one report (a ProfScope that
    spans two launches, e.g. enc_grad_simt = partial + reduce) the DRAM bytes are their sum."""
    out = page(rep, "raw")
    rows = [r for r in csv.reader(out.splitlines()) if r]
    h, units, vals = rows[0], rows[1], rows[2]
    m = {k: (vals[h.index(k)], units[h.index(k)]) for k in KEYS if k in h}
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        if k in h and len(rows) > 3:
            tot = sum(to_si(r[h.index(k)], units[h.index(k)]) or 0.0 for r in rows[2:] if len(r) == len(h))
            m[k] = (repr(tot), "byte")
    names = [r[h.index("Kernel Name")] for r in rows[2:] if len(r) == len(h)]
    return m, " + ".join(names)


def to_si(v, u):
    try:
        return float(v) * SCALE.get(u, 1.0)
    except ValueError:
        return None


def main():
    rnd, launches = sys.argv[1], sys.argv[2]
    reps = [a.split("=", 1) for a in sys.argv[3:]]
    lines = [f"# {rnd} ncu evidence", "",
             "Captured with `ncu --set full --clock-control none --import-source on` on one B200 "
             "(one kernel per report, after the same command exited 0 without ncu). Times under ncu are "
             "cold-cache and serialised: compare shares, not absolutes.", ""]
    traffic = {}
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(path):
        traffic = json.load(open(path))
    for name, rep in reps:
        m, kname = raw(rep)
        lines += [f"## {name}", "", f"Kernel: `{kname[:140]}`", "", "| metric | value | unit |", "|---|---|---|"]
        for k in KEYS:
            if k in m:
                lines.append(f"| {k} | {m[k][0]} | {m[k][1]} |")
        rd = to_si(*m["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in m else None
        wr = to_si(*m["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in m else None
        if rd is not None and wr is not None:
            traffic[name] = rd + wr
            lines += ["", f"DRAM traffic per launch: {rd + wr:.4g} B (read {rd:.4g}, write {wr:.4g})"]
        lines.append("")
    # kernel shares from the launch list ("-": none)
    rows = list(csv.reader(open(launches))) if launches != "-" else []
    hdr = None
    per = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            nm = d["Kernel Name"].split("(")[0].replace("void ", "")
            t = to_si(d["Metric Value"], d["Metric Unit"]) or 0.0
            per[nm] += t
            cnt[nm] += 1
    tot = sum(per.values()) or 1.0
    if rows:
        lines += [f"## Launch list ({os.path.basename(launches)}): share of device time", "",
                  "| kernel | launches | total (us) | share |", "|---|---|---|---|"]
    for nm, t in sorted(per.items(), key=lambda x: -x[1])[:25]:
        lines.append(f"| `{nm[:80]}` | {cnt[nm]} | {t * 1e6:.1f} | {100 * t / tot:.1f}% |")
    with open(os.path.join(ROOT, "profiles", f"{rnd}_ncu_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(path, "w") as f:
        json.dump(traffic, f, indent=1, sort_keys=True)
    print("\n".join(lines[:60]))


if __name__ == "__main__":
    main()
