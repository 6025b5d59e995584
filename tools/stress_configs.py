"""Full-size configs c1, c3, c4 (and c2 at two targets) on the device against the
oracle: ranks, container size within 1 %, reconstruction RE within 1 % of the
oracle's (both decoded by the device decompressor), timings."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_2107_01384_b200 as tcb  # noqa: E402
import synth  # noqa: E402

cases = [("c1", 1e-3), ("c2", 1e-4), ("c2", 1e-6), ("c3", 1e-3), ("c4", 1e-3)]
for cfg, re in cases:
    x = synth.make(cfg)
    src = tcb.SourceBuffer.from_array(x)
    for _ in range(2):
        r = tcb.compress(src, tcb.Params(target_re=re))
    t0 = time.perf_counter()
    r = tcb.compress(src, tcb.Params(target_re=re))
    dt = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter()
    o = oracle.compress(x, target_re=re)
    to = (time.perf_counter() - t0) * 1e3
    xd = x.astype(np.float64)
    nx = float((xd * xd).sum())
    y = tcb.decompress(r.container).to_array().astype(np.float64)
    yo = tcb.decompress(o.container).to_array().astype(np.float64)
    re_g = float(np.sqrt(((y - xd) ** 2).sum() / nx))
    re_o = float(np.sqrt(((yo - xd) ** 2).sum() / nx))
    ok = (r.ranks == o.ranks and abs(len(r.container) - len(o.container)) <= 0.01 * len(o.container)
          and re_g <= re * 1.05 and abs(re_g - re_o) <= 0.01 * re_o + 1e-15)
    print(f"{cfg} re={re:g}: ranks {r.ranks} vs {o.ranks}, bytes {len(r.container)} vs {len(o.container)}, "
          f"RE {re_g:.4e} vs {re_o:.4e}, gpu {dt:.1f} ms, oracle {to:.0f} ms -> {'OK' if ok else 'MISMATCH'}",
          flush=True)
