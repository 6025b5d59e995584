"""Time the device range coder on one long synthetic symbol stream (encode_symbols path)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2107_01384_b200 as tcb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
rng = np.random.default_rng(0)
syms = (rng.geometric(0.3, n) - 1).astype(np.uint64)
for it in range(3):
    t0 = time.perf_counter()
    out = tcb.encode_symbols(0, syms)
    dt = time.perf_counter() - t0
    print(f"n={n} bytes={len(out)} {dt * 1e3:.1f} ms ({dt / n * 1e9:.1f} ns/symbol)", flush=True)
