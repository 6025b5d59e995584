"""Summarise a timeline.json written by tools/timeline.py: kernels by wall time and
the main stream's sequence (segments over TL_MIN_US, default 1500 us)."""
import json
import os
import re
import sys
from collections import defaultdict

ev = json.load(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/timeline.json"))


def nm(s):
    s = s.replace("void ", "")
    s = re.sub(r"\(anonymous namespace\)::", "", s)
    s = s.split("(")[0]
    return s.split("::")[-1][:50] if "::" in s else s[:50]


agg = defaultdict(lambda: [0, 0.0])
for a, b, n, st in ev:
    k = nm(n)
    agg[k][0] += 1
    agg[k][1] += b - a
for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
    print(f"{k:50s} x{c:4d} {v / 1e3:8.2f}")
cnt = defaultdict(int)
for e in ev:
    cnt[e[3]] += 1
main = max(cnt, key=cnt.get)
for st in sorted(cnt):
    seq = [(a, b, nm(n)) for a, b, n, s in ev if s == st]
    out = []
    for a, b, n in seq:
        if out and out[-1][2] == n and a - out[-1][1] < 2000:
            out[-1][1] = b
            out[-1][3] += 1
        else:
            out.append([a, b, n, 1])
    print("stream", st, "(main)" if st == main else "", len(seq))
    for a, b, n, c in out:
        if b - a > float(os.environ.get("TL_MIN_US", 1500)):
            print(f"   {a / 1e3:7.1f}-{b / 1e3:7.1f} {n} x{c}")
