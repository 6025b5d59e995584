"""compute-sanitizer driver: one seeded compress + device decompress of a given
shape (no warm-up), with the reconstruction error checked, so memcheck /
racecheck / initcheck see every kernel of the path once.

  compute-sanitizer --tool memcheck python tools/sanitize_case.py 64 64 64 1e-3 float32 blobs
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2107_01384_b200 as tcb  # noqa: E402
import synth  # noqa: E402

shape = tuple(int(v) for v in sys.argv[1:4])
re = float(sys.argv[4])
dtype = np.dtype(sys.argv[5] if len(sys.argv) > 5 else "float32")
kind = sys.argv[6] if len(sys.argv) > 6 else "blobs"
x = synth.small(kind, shape, seed=1, dtype=dtype)
res = tcb.compress(tcb.SourceBuffer.from_array(x), tcb.Params(target_re=re))
y = tcb.decompress_tensor(res.container).reshape(shape)
xd = x.astype(np.float64)
err = float(np.sqrt(((y.astype(np.float64) - xd) ** 2).sum() / (xd ** 2).sum()))
print("shape", shape, "ranks", res.ranks, "bytes", len(res.container), "re", err, "launches", tcb.kernel_launches())
assert err <= 1.05 * re, err
