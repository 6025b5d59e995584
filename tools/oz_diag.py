"""Diagnostics: Ozaki TTM error pattern and c5 truncation SSE with / without the INT8 path."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2107_01384_b200 as tcb
from paper_2107_01384_b200 import shard
import synth

ops = shard.DeviceOps()
g = torch.Generator(device="cuda").manual_seed(2)
for rows, cols, r in [(200, 30000, 70), (1024, 50000, 650)]:
    b = torch.randn(rows, cols, dtype=torch.float64, device="cuda", generator=g)
    u = torch.linalg.qr(torch.randn(rows, r, dtype=torch.float64, device="cuda", generator=g))[0]
    out = ops.ttm_ozaki(b, u)
    ref = b.t() @ u
    err = (out - ref).abs()
    bound = torch.outer(b.norm(dim=0), u.norm(dim=0))
    rel = err / bound
    print(rows, cols, r, "max rel", float(rel.max()), "mean rel", float(rel.mean()),
          "mean signed (out-ref)/|ref|", float(((out - ref) * ref.sign()).mean() / ref.abs().mean()),
          "energy ratio", float((out * out).sum() / (ref * ref).sum()) - 1.0, flush=True)
    i = int(rel.argmax())
    print("  worst at", divmod(i, r), float(out.view(-1)[i]), float(ref.view(-1)[i]), flush=True)
    G = ops.gram_ozaki(b)
    Gr = b @ b.t()
    print("  gram energy-ish: trace diff", float(torch.trace(G) - torch.trace(Gr)),
          "offdiag max rel", float(((G - Gr).abs() / torch.outer(b.norm(dim=1), b.norm(dim=1))).max()), flush=True)
x = synth.grf_torch(n=1024, kmax=341, seed=0)
r = tcb.compress_device(x.data_ptr(), x.numel() * 4, tcb.Dtype.float32, list(x.shape), tcb.Params(target_re=1e-2))
print("c5 default: ranks", r.ranks, "trunc", r.estimate.truncation_sse, "bytes", len(r.container), flush=True)
