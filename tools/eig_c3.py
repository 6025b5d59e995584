"""Time the full eigensolver (values + r vectors) on c3's mode Grams, with the
device per-stage timer split (TCB_TRACE for host walls)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2107_01384_b200 as tcb  # noqa: E402
import synth  # noqa: E402

x = synth.make("c3").astype(np.float64)
for mode, r in ((1, 481), (2, 479)):
    b = np.moveaxis(x, mode, 0).reshape(x.shape[mode], -1)
    g = tcb.gram(b)
    for _ in range(2):
        tcb.eig(g, r)
    t0 = time.perf_counter()
    ev, v = tcb.eig(g, r)
    dt = (time.perf_counter() - t0) * 1e3
    ref = np.linalg.eigvalsh(g)[::-1]
    print(f"mode {mode}: n={g.shape[0]} r={r}: {dt:.1f} ms; eig rel err {np.max(np.abs(ev - ref)) / ref[0]:.2e}; "
          f"lambda_r/lambda_0 {ref[r - 1] / ref[0]:.2e}", flush=True)
