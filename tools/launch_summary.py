"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].replace("void ", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    name = name.split("(")[0].split("<")[0].split("::")[-1] or name
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':42s} {'launches':>8s} {'us':>10s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:42s} {v[0]:8d} {v[1]:10.1f} {100 * v[1] / tot:5.1f}%")
print(f"{'total':42s} {sum(v[0] for v in agg.values()):8d} {tot:10.1f}")
