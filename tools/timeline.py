"""Kernel timeline of one compress (torch.profiler / CUPTI sees the library's
launches on every stream): per-stream busy time, the span, and the top kernels
by wall time. Usage: python tools/timeline.py [re] [n]  (c5 by default)."""
import json
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2107_01384_b200 as tcb  # noqa: E402
import synth  # noqa: E402

re = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
x = synth.grf_torch(n=n, kmax=n // 3)
prm = tcb.Params(target_re=re)
for _ in range(2):
    r = tcb.compress_device(x.data_ptr(), x.numel() * 4, tcb.Dtype.float32, list(x.shape), prm)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    r = tcb.compress_device(x.data_ptr(), x.numel() * 4, tcb.Dtype.float32, list(x.shape), prm)
    torch.cuda.synchronize()
evs = []
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        evs.append((e.time_range.start, e.time_range.end, e.name, getattr(e, "device_resource_id", -1)))
evs.sort()
t0 = evs[0][0]
out = os.environ.get("TL_OUT", "gpurun_out/timeline.json")
with open(out, "w") as f:
    json.dump([[a - t0, b - t0, nm[:80], st] for a, b, nm, st in evs], f)
per_stream = defaultdict(float)
per_name = defaultdict(lambda: [0, 0.0])
for a, b, nm, st in evs:
    per_stream[st] += b - a
    k = nm.split("(")[0].split("<")[0][:60]
    per_name[k][0] += 1
    per_name[k][1] += b - a
span = evs[-1][1] - t0
print(f"compress n={n} re={re}: {len(evs)} device events, span {span / 1e3:.1f} ms, times {r.times}")
for st, v in sorted(per_stream.items(), key=lambda kv: -kv[1]):
    print(f"  stream {st}: busy {v / 1e3:.1f} ms")
# union of busy intervals (GPU active time)
busy, cur_a, cur_b = 0.0, None, None
for a, b, _, _ in evs:
    if cur_b is None or a > cur_b:
        if cur_b is not None:
            busy += cur_b - cur_a
        cur_a, cur_b = a, b
    else:
        cur_b = max(cur_b, b)
busy += cur_b - cur_a
print(f"  GPU busy (union) {busy / 1e3:.1f} ms, idle {(span - busy) / 1e3:.1f} ms")
for k, (c, v) in sorted(per_name.items(), key=lambda kv: -kv[1][1])[:40]:
    print(f"  {k:60s} x{c:5d} {v / 1e3:9.2f} ms")
# coarse timeline: 10 ms bins, the dominant kernel per bin
bins = defaultdict(lambda: defaultdict(float))
for a, b, nm, st in evs:
    k = nm.split("(")[0].split("<")[0][:30]
    t = a
    while t < b:
        bi = int((t - t0) // 10000)
        e = min(b, t0 + (bi + 1) * 10000)
        bins[bi][k] += e - t
        t = e
for bi in sorted(bins):
    top = sorted(bins[bi].items(), key=lambda kv: -kv[1])[:3]
    print(f"  {bi * 10:5d} ms: " + ", ".join(f"{k} {v / 1e3:.1f}" for k, v in top))
