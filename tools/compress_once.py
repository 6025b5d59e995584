"""Profiling driver: W warm-up + K compress calls of one config on cuda:0."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2107_01384_b200 as tcb  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--re", type=float, default=1e-4)
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--steps", type=int, default=1)
a = ap.parse_args()
x = synth.make(a.config)
src = tcb.SourceBuffer.from_array(x)
for i in range(a.warmup + a.steps):
    r = tcb.compress(src, tcb.Params(target_re=a.re))
print("ranks", r.ranks, "bytes", len(r.container), "lp", r.core_last_plane, "times", r.times)
