"""Oracle fixtures for c5 (1024^3 fp32 GRF, BASELINE configs[4]) at RE 1e-2 and
1e-3: one oracle/ compress + decompress per RE takes minutes of CPU time, too long
for the test suite, so tests/test_gpu_configs.py checks the device path against
these numbers instead.  Run on a GPU box (the input is the seeded torch-FFT
generator on the GPU, copied to the host for the oracle):

    python tests/golden/make_c5_fixtures.py [RE ...]  ->  tests/golden/c5_fixtures.json

(each RE takes ~10 minutes; the JSON is updated after every case)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402


def _save(path, out):
    with open(path, "w") as f:
        json.dump(out, f, indent=1)


def main(res):
    import torch

    t_start = time.perf_counter()
    seed = 0
    x = synth.grf_torch(n=1024, kmax=341, seed=seed)
    xs = x.double()
    checksum = [float(xs.sum()), float((xs * xs).sum()), float(xs[::97, ::89, ::83].sum())]
    del xs
    xh = x.cpu().numpy()
    path = os.path.join(ROOT, "tests", "golden", "c5_fixtures.json")
    out = json.load(open(path)) if os.path.exists(path) else {"cases": {}}
    out.update({"config": "c5: 1024^3 fp32 GRF E(k)~k^-5/3 (k<=341), synth.grf_torch(seed=0)", "seed": seed,
                "input_checksum": checksum, "oracle_threads": oracle.threads()})
    print(f"input ready ({time.perf_counter() - t_start:.1f} s), oracle threads {oracle.threads()}", flush=True)
    xd = x.double()
    den = float((xd * xd).sum())
    for re in res:
        t0 = time.perf_counter()
        info = oracle.compress(xh, target_re=re)
        t1 = time.perf_counter()
        case = {"ranks": list(info.ranks), "container_bytes": len(info.container),
                "truncation_sse": info.truncation_sse, "oracle_compress_s": t1 - t0}
        out["norm_sq"] = info.norm_sq
        # the oracle container's RE through the device decoder first (decoder parity is
        # pinned separately: tests/test_gpu_decompress.py), then through the oracle's own
        import paper_2107_01384_b200 as tcb

        buf = torch.empty(x.numel() * 4, dtype=torch.uint8, device="cuda")
        tcb.decompress_device(info.container, buf.data_ptr(), buf.numel())
        y = buf.view(torch.float32).view(x.shape).double()
        case["re_device_decoder"] = float(torch.sqrt(((y - xd) ** 2).sum() / den))
        del y, buf
        out["cases"][f"{re:g}"] = case
        _save(path, out)
        print(re, case, flush=True)
        y = oracle.decompress(info.container, xh.shape)
        case["re"] = float(np.sqrt(((y - xh.astype(np.float64)) ** 2).sum() / den))
        case["oracle_decompress_s"] = time.perf_counter() - t1
        del y
        _save(path, out)
        print(re, case, flush=True)


if __name__ == "__main__":
    main([float(v) for v in sys.argv[1:]] or [1e-2, 1e-3])
