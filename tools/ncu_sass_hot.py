"""Top SASS instructions by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
h = next(r for r in rows if r and r[0] == "Address")
hi = rows.index(h)
si = h.index("Warp Stall Sampling (All Samples)")
stall = [(i, c) for i, c in enumerate(h) if c.startswith("stall_")]
body = []
for r in rows[hi + 1:]:  # first kernel's section only
    if r and r[0] in ("Address", "Kernel Name"):
        break
    if len(r) == len(h):
        body.append(r)
tot = sum(int(r[si]) for r in body)
print(f"total samples {tot}")
for n, r in enumerate(body):
    r.append(n)
for r in sorted(body, key=lambda r: -int(r[si]))[:top]:
    reasons = sorted(((int(r[i]) if r[i].isdigit() else 0, c[6:]) for i, c in stall), reverse=True)[:2]
    rs = " ".join(f"{c}:{v}" for v, c in reasons if v)
    print(f"{r[-1]:5d} {int(r[si]):6d} {100 * int(r[si]) / tot:5.1f}%  {r[1].strip()[:60]:60s} {rs}")
