"""Time the Ozaki Gram / TTM (tcgen05 path, or TCB_OZAKI_LT=1) on c5's mode-0 shapes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2107_01384_b200 import shard  # noqa: E402

rows, cols, r = 1024, 1 << 20, 650
if len(sys.argv) > 1:
    rows, cols, r = (int(v) for v in sys.argv[1:4])
ops = shard.DeviceOps()
x = torch.randn(rows, cols, dtype=torch.float64, device="cuda").float().double()
u = torch.linalg.qr(torch.randn(rows, r, dtype=torch.float64, device="cuda"))[0]
for name, fn, ops_int8 in [("gram", lambda: ops.gram_ozaki(x), 15.0 * rows * (rows + 1) * cols),
                           ("ttm", lambda: ops.ttm_ozaki(x, u), 15.0 * 2 * rows * cols * r)]:
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    t = min(ts)
    print(f"{name} {rows}x{cols} r={r}: {t:.2f} ms (incl. split/combine), {ops_int8 / t / 1e9:.0f} int8 TOP/s "
          f"algorithmic", flush=True)
if os.environ.get("OZ_PROF"):
    from torch.profiler import ProfilerActivity, profile

    for name, fn in [("gram", lambda: ops.gram_ozaki(x)), ("ttm", lambda: ops.ttm_ozaki(x, u))]:
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            fn()
            torch.cuda.synchronize()
        for e in prof.key_averages():
            if e.device_time_total > 50:
                print(f"  {name}: {e.key[:70]:70s} {e.device_time_total / 1e3:8.2f} ms x{e.count}")
