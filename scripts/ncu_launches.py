"""Per-kernel summary of an ncu launch list (`--metrics gpu__time_duration.sum --csv`), grouped by
kernel name and grid size (launches of different levels / frame counts have different grids).

    python scripts/ncu_launches.py gpurun_out/launches.csv > profiles/rNN_launches.txt
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
gi = h.index("Grid Size") if "Grid Size" in h else None
d = defaultdict(list)
order = []
for r in rows[hi + 1:]:
    key = (r[ki].split("(")[0][:48], r[gi] if gi is not None else "")
    if key not in d:
        order.append(key)
    scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1e-3)
    d[key].append(float(r[vi].replace(",", "")) * scale)
print(f"{'launches':>8} {'mean us':>10} {'min us':>10}  kernel / grid")
for k in order:
    v = d[k]
    print(f"{len(v):8d} {sum(v) / len(v):10.1f} {min(v):10.1f}  {k[0]} {k[1]}")
