"""Read one page of an ncu report as CSV text: from the .ncu-rep if it is here, else from the CSV
exports tools/ncu_export.sh writes next to it on the GPU box (<rep>.<page>.csv.gz), so large
reports need not travel back."""
import gzip
import os
import subprocess


def page(rep, name, extra=()):
    if os.path.exists(rep):
        return subprocess.run(["ncu", "-i", rep, "--page", name, "--csv", *extra], capture_output=True,
                              text=True).stdout
    base = rep[:-len(".ncu-rep")] if rep.endswith(".ncu-rep") else rep
    path = f"{base}.{name}.csv.gz"
    with gzip.open(path, "rt") as f:
        return f.read()
