"""Profiling driver: compress c2 once, then W warm-up + K decompress calls."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

import paper_2107_01384_b200 as tcb  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--re", type=float, default=1e-4)
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--steps", type=int, default=5)
a = ap.parse_args()
x = synth.make(a.config)
c = tcb.compress(tcb.SourceBuffer.from_array(x), tcb.Params(target_re=a.re)).container
for _ in range(a.warmup):
    tcb.decompress(c)
ts = []
for _ in range(a.steps):
    t0 = time.perf_counter()
    r = tcb.decompress(c)
    ts.append((time.perf_counter() - t0) * 1e3)
y = r.to_array()
print("decompress ms", [round(t, 3) for t in ts], "device ms", round(r.total_ms, 3),
      "RE", float(np.sqrt(((y - x) ** 2).sum() / (x ** 2).sum())))
