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


def main(res):
    seed = 0
    x = synth.grf_torch(n=1024, kmax=341, seed=seed)
    xs = x.double()
    checksum = [float(xs.sum()), float((xs * xs).sum()), float(xs[::97, ::89, ::83].sum())]
    del xs
    xh = x.cpu().numpy()
    del x
    path = os.path.join(ROOT, "tests", "golden", "c5_fixtures.json")
    out = json.load(open(path)) if os.path.exists(path) else {"cases": {}}
    out.update({"config": "c5: 1024^3 fp32 GRF E(k)~k^-5/3 (k<=341), synth.grf_torch(seed=0)", "seed": seed,
                "input_checksum": checksum, "oracle_threads": oracle.threads()})
    xd = xh.astype(np.float64)
    den = float((xd * xd).sum())
    for re in res:
        t0 = time.perf_counter()
        info = oracle.compress(xh, target_re=re)
        t1 = time.perf_counter()
        y = oracle.decompress(info.container, xh.shape)
        e = float(np.sqrt(((y - xd) ** 2).sum() / den))
        out["norm_sq"] = info.norm_sq
        out["cases"][f"{re:g}"] = {"ranks": list(info.ranks), "container_bytes": len(info.container),
                                   "truncation_sse": info.truncation_sse, "re": e,
                                   "oracle_compress_s": t1 - t0}
        print(re, out["cases"][f"{re:g}"], flush=True)
        del y
        with open(path, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main([float(v) for v in sys.argv[1:]] or [1e-2, 1e-3])
