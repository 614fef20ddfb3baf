"""Print the `details` page of one kernel (by ID) of an ncu report, section by section.

  python tools/ncu_details.py <report.ncu-rep> <ID> [section-regex]
"""
import csv, re, subprocess, sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.abspath(__file__)))
from ncu_page import page  # noqa: E402
rep, kid = sys.argv[1], sys.argv[2]
pat = re.compile(sys.argv[3] if len(sys.argv) > 3 else ".")
out = page(rep, "details")
rows = list(csv.reader(out.splitlines()))
h = rows[0]
I = {k: h.index(k) for k in ("ID", "Kernel Name", "Section Name", "Metric Name", "Metric Unit", "Metric Value")}
name = None
for r in rows[1:]:
    if len(r) <= I["Metric Value"] or r[I["ID"]] != kid:
        continue
    if name is None:
        name = r[I["Kernel Name"]]
        print(name[:150])
    if pat.search(r[I["Section Name"]]) and r[I["Metric Name"]]:
        print(f"  {r[I['Section Name']][:28]:28s} {r[I['Metric Name']][:52]:52s} {r[I['Metric Value']]:>14s} {r[I['Metric Unit']]}")
