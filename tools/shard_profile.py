"""Wall time of each DeviceOps call inside one sharded compress (world size 1)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2107_01384_b200 as tcb  # noqa: E402
from paper_2107_01384_b200 import shard  # noqa: E402


class Timed(shard.DeviceOps):
    log = []

    def __getattribute__(self, name):
        f = super().__getattribute__(name)
        if name.startswith("_") or not callable(f):
            return f

        def w(*a, **k):
            torch.cuda.synchronize()
            t = time.perf_counter()
            r = f(*a, **k)
            torch.cuda.synchronize()
            Timed.log.append((name, 1e3 * (time.perf_counter() - t)))
            return r
        return w


x = torch.from_numpy(bench.c2_slab(1, 0)).cuda()
p = tcb.Params(target_re=1e-4)
for _ in range(3):
    shard.compress_sharded(x, [256, 256, 256], tcb.Dtype.float64, p, ops=Timed())
Timed.log.clear()
torch.cuda.synchronize()
t0 = time.perf_counter()
shard.compress_sharded(x, [256, 256, 256], tcb.Dtype.float64, p, ops=Timed())
torch.cuda.synchronize()
tot = 1e3 * (time.perf_counter() - t0)
for n, ms in Timed.log:
    print(f"{n:18s} {ms:7.3f} ms")
print(f"{'total':18s} {tot:7.3f} ms (calls {sum(ms for _, ms in Timed.log):.3f})")
