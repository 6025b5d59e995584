"""Per-step times of the end-to-end C-ABI call (tcb_compress from pinned host
memory) on c5, with the library's phase times, to see where outliers come from.
Usage: python tools/e2e_steps.py [steps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2107_01384_b200 as tcb  # noqa: E402
import synth  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 12
x = synth.grf_torch(n=1024, kmax=341)
host = x.cpu().pin_memory()
if os.environ.get("E2E_FREE_DEV"):
    del x
    torch.cuda.empty_cache()
prm = tcb.Params(target_re=1e-2)
src = tcb.SourceBuffer(memoryview(host.numpy()).cast("B"), tcb.Dtype.float32, [1024, 1024, 1024])
for i in range(steps):
    torch.cuda.synchronize()
    t = time.perf_counter()
    raw = tcb.compress_raw(src, prm)
    dt = time.perf_counter() - t
    tm = raw.times
    print(f"step {i}: {dt * 1e3:7.1f} ms  sthosvd {tm.sthosvd_ms:6.1f} quant {tm.quantize_ms:5.1f} core {tm.core_encode_ms:6.1f} "
          f"factor {tm.factor_encode_ms:6.1f} ser {tm.serialize_ms:5.1f} total {tm.total_ms:6.1f}", flush=True)
    tcb.free_raw(raw)
free, total = torch.cuda.mem_get_info()
print(f"device memory in use after the steps (pool included): {(total - free) / 2**30:.1f} GiB of {total / 2**30:.1f}")
