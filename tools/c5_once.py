"""c5 (1024^3 fp32 GRF, generated on the GPU) through tcb_compress_device, RE check on the device."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2107_01384_b200 as tcb  # noqa: E402
import synth  # noqa: E402

re = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
x = synth.grf_torch(n=n, kmax=n // 3)
assert x.dtype == torch.float32 and x.is_cuda
iters = int(os.environ.get('C5_ITERS', '2'))
prof = os.environ.get('C5_PROFILE')  # ncu --profile-from-start off: only the last compress is captured
for it in range(iters):
    torch.cuda.synchronize()
    if prof and it == iters - 1:
        torch.cuda.profiler.start()
    t0 = time.perf_counter()
    r = tcb.compress_device(x.data_ptr(), x.numel() * 4, tcb.Dtype.float32, list(x.shape), tcb.Params(target_re=re))
    torch.cuda.synchronize()
    if prof and it == iters - 1:
        torch.cuda.profiler.stop()
    dt = time.perf_counter() - t0
    print(f"c5 n={n} re={re:g}: {dt * 1e3:.1f} ms, ranks {r.ranks}, bytes {len(r.container)}, "
          f"factor {r.compression_factor():.1f}, times {r.times}", flush=True)
if os.environ.get('C5_NO_DEC'):
    sys.exit(0)
out = torch.empty(x.numel() * 4, dtype=torch.uint8, device="cuda")
tcb.decompress_device(r.container, out.data_ptr(), out.numel())
y = out.view(torch.float32).view(x.shape).double()
xd = x.double()
print("achieved RE", float(torch.sqrt(((y - xd) ** 2).sum() / (xd * xd).sum())))
