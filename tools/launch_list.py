"""Print the launches of an ncu --csv launch list whose kernel name matches a pattern, in order."""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
pat = re.compile(sys.argv[2] if len(sys.argv) > 2 else ".")
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
H = rows[h]
ki, vi, ui = H.index("Kernel Name"), H.index("Metric Value"), H.index("Metric Unit")
gi = H.index("Grid Size") if "Grid Size" in H else None
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
for r in rows[h + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].replace("void ", "").replace("(anonymous namespace)::", "").split("(")[0]
    name = re.sub(r"tcb::|<unnamed>::|_GLOBAL__N_\w+::", "", name)
    if pat.search(name):
        us = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        print(f"{name[:48]:48s} {us:12.1f} us  grid {r[gi] if gi is not None else ''}")
