"""Every compiled SYRK shape (gemm.cu kSyrk, selected by TCB_GRAM_VARIANT) and
the diagonal slab balancing (TCB_GRAM_DIAG_BALANCE) against a plain fp64
reference on the edge shapes: one partial tile (no off-diagonal tiles), row
counts that cut a diagonal tile, odd column counts (8-byte loads), and a
split-K plan with many splits.  The plan is chosen once per process, so each
setting runs in a child process."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHAPES = [(1, 5), (20, 33), (64, 64), (100, 301), (130, 257), (200, 4096), (256, 20000),
          (700, 3001), (1024, 8192)]  # multi-tile triangular index math and split plan (c5's 1024-row modes)

CHILD = r"""
import json, sys
import numpy as np
sys.path.insert(0, %r)
import paper_2107_01384_b200 as pkg
out = []
for rows, cols in %r:
    b = np.random.default_rng(rows * 7919 + cols).standard_normal((rows, cols))
    g = pkg.gram(b)
    ref = b @ b.T
    out.append(float(np.abs(g - ref).max() / np.abs(ref).max()))
    assert np.array_equal(g, g.T)
print(json.dumps(out))
"""


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", CHILD % (ROOT, SHAPES)], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
@pytest.mark.parametrize("variant", range(10))
@pytest.mark.parametrize("balance", ["0", "1"])
def test_gram_variant_matches_fp64(variant, balance):
    errs = _run({"TCB_GRAM_VARIANT": str(variant), "TCB_GRAM_DIAG_BALANCE": balance})
    # fp64 accumulation over up to 20000 terms: relative to max |G|
    assert max(errs) < 1e-13, dict(zip(map(str, SHAPES), errs))
