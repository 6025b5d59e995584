"""Regenerate tests/golden/golden.json from the REFERENCE'S OWN code.

Every vector below is produced by oracle/_ref/libtucomp_ref.so, i.e. the
reference's core_codec.cpp / entropy.cpp / error_model.cpp / container.cpp /
kernels*.cpp compiled verbatim from /root/reference/proj/src by
oracle/ref/build_ref.sh.  Only inputs are synthetic (seeded numpy).  Run here
(where /root/reference exists):  python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle.ref as R  # noqa: E402


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def core_like(shape, seed, decay):
    rng = np.random.default_rng(seed)
    idx = np.indices(shape).sum(0).astype(np.float64)
    return rng.standard_normal(shape) * np.exp(-decay * idx / idx.max())


def main():
    if not R.available():
        raise SystemExit("oracle/_ref not built: run oracle/ref/build_ref.sh first")
    out = {"generator": "tests/golden/make_golden.py", "source": "verbatim reference integer TUs (oracle/_ref)",
           "symbols": [], "encode": [], "quantize": [], "sum_squares": []}
    rng = np.random.default_rng(2024)
    for case, syms in enumerate([
        [],
        [0],
        [5, 5, 5, 5],
        list(rng.geometric(0.3, 200) - 1),
        list(np.concatenate([rng.geometric(0.02, 2000) - 1, rng.integers(0, 2 ** 32 - 1, 40)])),
        [2 ** 32 - 1, 0, 2 ** 32 - 1, 1],
    ]):
        syms = np.asarray(syms, np.uint64)
        for coder in (0, 1):
            b = R.encode_symbols(coder, syms)
            out["symbols"].append({"case": case, "coder": coder, "symbols": [int(v) for v in syms],
                                   "bytes": b.hex()})
    for seed, shape, decay in [(1, (12, 13, 14), 5.0), (2, (20, 21, 22), 7.0), (3, (9, 40, 70), 4.0)]:
        core = core_like(shape, seed, decay)
        mag, neg, k, zero, sn = R.quantize(core)
        out["quantize"].append({"seed": seed, "shape": list(shape), "decay": decay, "k": k, "zero": zero,
                                "mag_sha": sha(mag.tobytes()), "neg_sha": sha(neg.tobytes()),
                                "slice_norms_hex": [[float(v).hex() for v in ax] for ax in sn]})
        tot = float((mag.astype(np.float64) ** 2).sum())
        for frac in (1e-1, 1e-4, 1e-8, 0.0):
            for coder in (0, 1):
                for split in (True, False):
                    s, lp, ach, dec = R.encode(mag, neg, tot * frac, coder=coder, split=split)
                    out["encode"].append({"seed": seed, "shape": list(shape), "decay": decay, "frac": frac,
                                          "coder": coder, "split": split, "fixed": -1, "last_plane": lp,
                                          "len": len(s), "sha": sha(s), "achieved_hex": float(ach).hex(),
                                          "dec_sha": sha(dec.tobytes())})
        for fixed in (60, 45, 30):
            s, lp, ach, dec = R.encode(mag, neg, 0.0, split=False, fixed_plane=fixed)
            out["encode"].append({"seed": seed, "shape": list(shape), "decay": decay, "frac": 0.0, "coder": 0,
                                  "split": False, "fixed": fixed, "last_plane": lp, "len": len(s), "sha": sha(s),
                                  "achieved_hex": float(ach).hex(), "dec_sha": sha(dec.tobytes())})
    for n in (0, 1, 7, 8, 9, 1000, 4097):
        x = np.random.default_rng(n).uniform(-3, 3, n)
        out["sum_squares"].append({"n": n, "dtype": "float64", "value_hex": float(R.sum_sq(x)).hex()})
        out["sum_squares"].append({"n": n, "dtype": "float32",
                                   "value_hex": float(R.sum_sq(x.astype(np.float32))).hex()})
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=0)
    print(f"wrote {path}: {len(out['symbols'])} symbol vectors, {len(out['encode'])} streams")


if __name__ == "__main__":
    main()
