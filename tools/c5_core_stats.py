"""msb histogram of c5's quantised core (per plane, per block): sizes the encoder's work."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2107_01384_b200 as tcb  # noqa: E402
import synth  # noqa: E402

re = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-2
x = synth.grf_torch(n=1024, kmax=341)
a = x.double().cpu().numpy()
del x
norm = float((a * a).sum())
st = tcb.sthosvd(a, 0.5 * re * re * norm)
del a
core = st["core"]
mag, neg, k, zero, sn = tcb.quantize(core)
msb = np.where(mag == 0, -1, np.floor(np.log2(np.maximum(mag, 1).astype(np.float64))).astype(np.int64))
# log2 of u64 in float64 may round up at 2^k - small: fix by comparing
fix = (msb >= 0) & (np.left_shift(np.uint64(1), msb.clip(0).astype(np.uint64)) > mag)
msb[fix] -= 1
hist = np.bincount(msb + 1, minlength=65)
n = mag.size
block = max(4096, -(-n // 64))
nb = -(-n // block)
per_block = {}
for p in range(63, 40, -1):
    c = (msb == p)
    per_block[p] = [int(c[b * block:(b + 1) * block].sum()) for b in range(nb)]
res = dict(n=int(n), k=int(k), ranks=st["ranks"], hist={str(i - 1): int(h) for i, h in enumerate(hist) if h},
           block=int(block), per_block_new=per_block)
with open("gpurun_out/c5_core_stats.json", "w") as f:
    json.dump(res, f)
print(json.dumps({k: v for k, v in res.items() if k != "per_block_new"}))
