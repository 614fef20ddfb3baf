"""Key metrics of the first kernel of an ncu report (speed of light, issue, occupancy, pipes).
  python tools/ncu_brief.py <report.ncu-rep>"""
import csv, subprocess, sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.abspath(__file__)))
from ncu_page import page  # noqa: E402
out = page(sys.argv[1], "details")
r = list(csv.reader(out.splitlines()))
h = r[0]
si, mi, vi, ui = h.index("Section Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
keep = ("Duration", "Issue Slots Busy", "Executed Ipc Active", "Achieved Active Warps Per SM", "DRAM Throughput",
        "Memory Throughput", "Eligible Warps Per Scheduler", "Registers Per Thread", "No Eligible",
        "Compute (SM) Throughput", "L2 Cache Throughput", "L1/TEX Cache Throughput", "Warp Cycles Per Issued Instruction")
seen = set()
for x in r[1:]:
    if len(x) > vi and x[mi] in keep and x[mi] not in seen:
        seen.add(x[mi])
        print(f"{x[mi][:40]:40s} {x[vi]:>12s} {x[ui]}")
raw = page(sys.argv[1], "raw")
rr = list(csv.reader(raw.splitlines()))
hh = rr[0]
want = ["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__inst_executed_pipe_tc_scope_2cta.sum", "gpu__time_duration.sum"]
for w in want:
    if w in hh:
        i = hh.index(w)
        print(f"{w:66s} {rr[2][i]:>14s} {rr[1][i]}")
