"""Evaluation (not the product path): fp64 Gram emulation on INT8 tensor cores
(Ozaki scheme I) for c5's mode-0 Gram, against the fp64 Gram.

  python tools/ozaki_eval.py [S ...]      (on a GPU box)

Each row of X (1024 x 1M, the c5 tensor's mode-0 unfolding) is scaled by a power
of two to [-1, 1) and split into S int8 digit slices (first slice 6 bits + sign,
then 7 bits each, every digit in [-64, 64]), so X = diag(2^e) sum_s 2^-w_s D_s
exactly up to the last slice's rounding.  G = X X^T is then the sum over slice
pairs (s, t) with s + t <= S + 1 of 2^-(w_s + w_t) D_s D_t^T: every product is an
int8 GEMM accumulated exactly in int32 (|digit| <= 64, so k-chunks of 2^19 terms
cannot overflow), converted to fp64 and scaled exactly.  The GEMMs here are
torch._int_mm (cuBLASLt IMMA) -- this measures what the tensor cores give, not a
hand-written kernel.  Reported per S: time of the S(S+1)/2 products + split +
accumulation, the fp64 DGEMM time, the Gram error relative to |x_i||x_j|, the
relative error of the top-650 eigenvalues, and the largest principal-angle sine
of the top-650 eigenspace (the c5 @ 1e-2 rank).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402

KCH = 1 << 19


def split(x64, S):
    """Row scale exponents and S int8 digit slices (row-major, K padded to a multiple of 8)."""
    amax = x64.abs().amax(dim=1).clamp_min(1e-300)
    e = torch.ceil(torch.log2(amax))
    r = x64 * torch.exp2(-e)[:, None]  # |r| <= 1
    ds = []
    w = []
    sh = 6
    acc = 0
    for s in range(S):
        acc += sh
        v = torch.round(r * (2.0 ** sh))
        ds.append(v.to(torch.int8))
        w.append(acc)
        r = r * (2.0 ** sh) - v  # exact: |r| <= 1/2
        sh = 7
    return e, ds, w


def ozaki_gram(x64, S):
    e, ds, w = split(x64, S)
    n, k = x64.shape
    g = torch.zeros(n, n, dtype=torch.float64, device=x64.device)
    for s in range(S):
        for t in range(S):
            if s + t > S - 1:
                continue
            acc = torch.zeros(n, n, dtype=torch.float64, device=x64.device)
            for k0 in range(0, k, KCH):
                a = ds[s][:, k0:k0 + KCH]
                b = ds[t][:, k0:k0 + KCH]
                acc += torch._int_mm(a, b.t()).double()
            g += acc * (2.0 ** -(w[s] + w[t]))
    sc = torch.exp2(e)
    return g * sc[:, None] * sc[None, :]


def timeit(fn, reps=3):
    out = None
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        out = fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return out, min(ts)


def main():
    Ss = [int(v) for v in sys.argv[1:]] or [4, 5, 6, 8]
    x = synth.grf_torch(n=1024, kmax=341, seed=0)
    x64 = x.double().reshape(1024, -1)
    del x
    g64, t64 = timeit(lambda: x64 @ x64.t())
    nrm = x64.norm(dim=1)
    ev, vec = torch.linalg.eigh(g64)
    ev, vec = ev.flip(0), vec.flip(1)
    r = 650
    print(f"fp64 DGEMM (cuBLAS, full 1024x1024x1M): {t64:.2f} ms = {2 * 1024 * 1024 * x64.shape[1] / t64 / 1e9:.1f} TF/s",
          flush=True)
    # raw int8 GEMM rate on one chunk
    a = torch.randint(-64, 65, (1024, KCH), dtype=torch.int8, device="cuda")
    _, ti = timeit(lambda: torch._int_mm(a, a.t()), reps=5)
    print(f"int8 GEMM 1024x1024x{KCH}: {ti:.3f} ms = {2 * 1024 * 1024 * KCH / ti / 1e9:.0f} TOP/s", flush=True)
    del a
    # the library's rate on a shape with enough output tiles for every SM
    a = torch.randint(-64, 65, (8192, 32768), dtype=torch.int8, device="cuda")
    b = torch.randint(-64, 65, (8192, 32768), dtype=torch.int8, device="cuda")
    _, ti = timeit(lambda: torch._int_mm(a, b.t()), reps=5)
    print(f"int8 GEMM 8192x8192x32768: {ti:.3f} ms = {2 * 8192 * 8192 * 32768 / ti / 1e9:.0f} TOP/s", flush=True)
    del a, b
    for S in Ss:
        g, t = timeit(lambda: ozaki_gram(x64, S), reps=2)
        err = ((g - g64).abs() / (nrm[:, None] * nrm[None, :])).max().item()
        eo, vo = torch.linalg.eigh(g)
        eo, vo = eo.flip(0), vo.flip(1)
        ere = ((eo[:r] - ev[:r]).abs() / ev[0]).max().item()
        sv = torch.linalg.svdvals(vec[:, :r].t() @ vo[:, :r])
        sine = float(torch.sqrt(torch.clamp(1 - sv.min() ** 2, min=0)))
        print(f"S={S}: {S * (S + 1) // 2} int8 products, {t:.2f} ms (incl. split + fp64 accumulation in torch); "
              f"max |dG|/(|x_i||x_j|) = {err:.2e}; top-{r} eigenvalue error / lambda_1 = {ere:.2e}; "
              f"top-{r} subspace sine = {sine:.2e}", flush=True)


if __name__ == "__main__":
    main()
