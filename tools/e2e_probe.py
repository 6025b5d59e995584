"""c5 end-to-end anatomy: raw pinned H2D rate, tcb.compress (host API) vs
compress_device, and the Python-side container copy."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2107_01384_b200 as tcb  # noqa: E402
import synth  # noqa: E402

x = synth.grf_torch(n=1024, kmax=341)
host = x.cpu().pin_memory()
dev = torch.empty_like(x)
for _ in range(3):
    dev.copy_(host, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(3):
    dev.copy_(host, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 3
print(f"pinned H2D 4 GiB: {dt * 1e3:.1f} ms = {x.numel() * 4 / dt / 1e9:.1f} GB/s", flush=True)
prm = tcb.Params(target_re=1e-2)
src = tcb.SourceBuffer(memoryview(host.numpy()).cast("B"), tcb.Dtype.float32, list(x.shape))
for i in range(4):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = tcb.compress(src, prm)
    t1 = time.perf_counter()
    rd = tcb.compress_device(x.data_ptr(), x.numel() * 4, tcb.Dtype.float32, list(x.shape), prm)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    raw = tcb.compress_device_raw(x.data_ptr(), x.numel() * 4, tcb.Dtype.float32, list(x.shape), prm)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    tcb.lib().tcb_free(raw.container)
    print(f"iter {i}: host API {1e3 * (t1 - t):.1f} ms, device API {1e3 * (t2 - t1):.1f} ms, "
          f"device raw (no bytes copy) {1e3 * (t3 - t2):.1f} ms, same {r.container == rd.container}, times {r.times}",
          flush=True)
