"""Time the SYRK kernel shapes (TCB_GRAM_VARIANT) on the c2 Gram shapes.

  python tools/gram_variants.py            # one process per variant
Prints per variant and shape: ms per Gram (CUDA-event stage time, kernel +
fixed-order reduction), algorithmic TF/s (rows*(rows+1)*cols flops), and the
max deviation from torch's fp64 A A^T relative to max |G|."""
import ctypes as C
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child():
    sys.path.insert(0, ROOT)
    import torch
    import paper_2107_01384_b200 as pkg
    lib = pkg.lib()
    out = {}
    for rows, cols in [(256, 65536), (256, 3584), (256, 182)]:
        g = torch.Generator(device="cuda").manual_seed(1)
        a = torch.randn(rows, cols, dtype=torch.float64, device="cuda", generator=g)
        gm = torch.empty(rows, rows, dtype=torch.float64, device="cuda")
        for _ in range(3):
            assert lib.tcb_dev_gram(C.c_void_p(a.data_ptr()), C.c_uint64(rows), C.c_uint64(cols),
                                    C.c_void_p(gm.data_ptr())) == 0
        torch.cuda.synchronize()
        lib.tcb_prof_enable(1)
        ms = (C.c_double * 11)()
        cnt = (C.c_uint64 * 11)()
        lib.tcb_prof_read(ms, cnt, 11)
        it = 20
        for _ in range(it):
            lib.tcb_dev_gram(C.c_void_p(a.data_ptr()), C.c_uint64(rows), C.c_uint64(cols), C.c_void_p(gm.data_ptr()))
        lib.tcb_prof_read(ms, cnt, 11)
        lib.tcb_prof_enable(0)
        t = ms[2] / it
        ref = a @ a.T
        err = float((gm - ref).abs().max() / ref.abs().max())
        out[f"{rows}x{cols}"] = {"ms": round(t, 4), "tflops": round(rows * (rows + 1) * cols / t / 1e9, 2),
                                  "err": err}
    print(json.dumps(out))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        child()
    else:
        for v in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
            env = dict(os.environ, TCB_GRAM_VARIANT=str(v))
            r = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True)
            print(v, r.stdout.strip() or r.stderr[-2000:], flush=True)
