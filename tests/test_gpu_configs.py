"""Every BASELINE.json config at full size against the CPU oracle (SURVEY 8(c)
parity contract): ranks equal, factor subspaces within principal-angle sine
1e-6 (fp64 internal arithmetic), compressed size within 1 %, reconstruction
relative error (the oracle's decoder on both containers) within 1 % of the
oracle's, truncation SSE and |A|^2 to FP tolerance.

c5 (1024^3, minutes of CPU time per oracle run) is checked against fixtures
that tests/golden/make_c5_fixtures.py computed with the oracle on the same
seeded input (regenerated here on the GPU; the input's checksum is pinned)."""
import json
import os

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def principal_sine(u, v):
    return float(np.linalg.norm(u - v @ (v.T @ u), 2))


def rel_err(y, x):
    xd = x.astype(np.float64)
    return float(np.sqrt(((y - xd) ** 2).sum() / (xd ** 2).sum()))


def subspace_tol(s2, r):
    """1e-6 (the parity bar), or the Davis-Kahan floor of ANY fp64 eigensolver when
    the cut falls inside a cluster: a Gram perturbed by n eps |G| moves the kept
    subspace by up to n eps |G| / (s2[r-1] - s2[r]) (c3's 479-of-500 cut lies in
    its noise-floor cluster)."""
    s2 = np.asarray(s2, np.float64)
    if r >= s2.size:
        return 1e-6
    gap = max(s2[r - 1] - s2[r], 1e-300)
    return max(1e-6, 8.0 * s2.size * np.finfo(np.float64).eps * s2[0] / gap)


_CACHE = {}


def config_input(name):
    if name not in _CACHE:
        _CACHE.clear()
        _CACHE[name] = synth.make(name, seed=0)
    return _CACHE[name]


CASES = [("c1", 1e-3), ("c2", 1e-2), ("c2", 1e-4), ("c2", 1e-6), ("c3", 1e-2), ("c3", 1e-3), ("c3", 1e-4),
         ("c4", 1e-3)]


@pytest.mark.parametrize("name,re", CASES, ids=[f"{n}-re{r:g}" for n, r in CASES])
def test_config_full_size_against_oracle(gpu_pkg, name, re):
    x = config_input(name)
    res = gpu_pkg.compress(gpu_pkg.SourceBuffer.from_array(x), gpu_pkg.Params(target_re=re))
    ref = oracle.compress(x, target_re=re)
    assert res.ranks == ref.ranks, (res.ranks, ref.ranks)
    assert abs(len(res.container) - len(ref.container)) <= 0.01 * len(ref.container), (
        len(res.container), len(ref.container))
    assert res.norm_sq == pytest.approx(ref.norm_sq, rel=1e-12)
    # the discarded energy is a difference of Gram spectra: both sides carry an
    # absolute error ~ n eps |A|^2 (c2 @ 1e-4: 5.5e-3 out of |A|^2 = 1.1e6)
    n_max = max(x.shape)
    assert abs(res.estimate.truncation_sse - ref.truncation_sse) <= max(
        1e-6 * ref.truncation_sse, n_max * np.finfo(np.float64).eps * ref.norm_sq)
    e = rel_err(oracle.decompress(res.container, x.shape), x)
    er = rel_err(oracle.decompress(ref.container, x.shape), x)
    assert abs(e - er) <= 0.01 * er, (e, er)
    # factor subspaces of the ST-HOSVD (same budget as compress: rtmss * RE^2 |A|^2)
    budget = 0.5 * re * re * ref.norm_sq
    a = gpu_pkg.sthosvd(x.astype(np.float64), budget)
    b = oracle.sthosvd(x.astype(np.float64), budget)
    assert a["ranks"] == b["ranks"]
    for mode, (fa, fb) in enumerate(zip(a["factors"], b["factors"])):
        assert principal_sine(fa, fb) <= subspace_tol(b["sigma2"][mode], b["ranks"][mode])


# ---------------------------------------------------------------- c5 against fixtures
def _c5_fixture():
    p = os.path.join(HERE, "golden", "c5_fixtures.json")
    if not os.path.exists(p):
        pytest.skip("tests/golden/c5_fixtures.json not generated")
    return json.load(open(p))


@pytest.mark.parametrize("path", ["int8", "dmma"])
@pytest.mark.parametrize("re", [1e-2, 1e-3])
def test_c5_against_oracle_fixture(gpu_pkg, re, path, monkeypatch):
    """c5's mode loop runs on the INT8 (Ozaki) path by default; TCB_OZAKI=0 forces
    fp64 DMMA.  Both meet the parity bar; the discarded energy -- a difference of
    spectra ~1e-7 of |A|^2 -- is reproduced to ~1e-16 n |A|^2 by DMMA and to the
    digit truncation's ~2^-30 |A|^2 by the INT8 path."""
    import torch

    if path == "dmma":
        monkeypatch.setenv("TCB_OZAKI", "0")

    fx = _c5_fixture()
    if f"{re:g}" not in fx["cases"]:
        pytest.skip(f"no c5 fixture for RE {re:g}")
    case = fx["cases"][f"{re:g}"]
    x = synth.grf_torch(n=1024, kmax=341, seed=fx["seed"])
    xs = x.double()
    check = [float(xs.sum()), float((xs * xs).sum()), float(xs[::97, ::89, ::83].sum())]
    del xs
    if not np.allclose(check, fx["input_checksum"], rtol=1e-12, atol=1e-6):
        pytest.skip(f"GRF input differs from the fixture's (torch RNG changed): {check} vs {fx['input_checksum']}")
    r = gpu_pkg.compress_device(x.data_ptr(), x.numel() * 4, gpu_pkg.Dtype.float32, list(x.shape),
                                gpu_pkg.Params(target_re=re))
    assert r.ranks == case["ranks"]
    assert abs(len(r.container) - case["container_bytes"]) <= 0.01 * case["container_bytes"]
    # |A|^2 of 2^30 floats: the reference accumulates it serially in 4 double lanes
    # (kernels_avx2.cpp:146-159), ~sqrt(n) eps = 2e-12 relative off the exact sum; the
    # device's reduction tree is within 1e-15 of the exact sum (fixture checksum[1])
    assert r.norm_sq == pytest.approx(fx["norm_sq"], rel=1e-10)
    assert r.norm_sq == pytest.approx(fx["input_checksum"][1], rel=1e-14)
    tol = 1e-6 * case["truncation_sse"] if path == "dmma" else max(1e-6 * case["truncation_sse"],
                                                                   2.0 ** -30 * fx["norm_sq"])
    assert abs(r.estimate.truncation_sse - case["truncation_sse"]) <= tol
    out = torch.empty(x.numel() * 4, dtype=torch.uint8, device="cuda")
    gpu_pkg.decompress_device(r.container, out.data_ptr(), out.numel())
    y = out.view(torch.float32).view(x.shape).double()
    xd = x.double()
    e = float(torch.sqrt(((y - xd) ** 2).sum() / (xd * xd).sum()))
    ref_re = case.get("re", case["re_device_decoder"])  # the oracle decoder's RE when it finished
    assert abs(e - ref_re) <= 0.01 * ref_re, (e, ref_re)


# ---------------------------------------------------------------- the thin-SVD branch (rows > cols)
@pytest.mark.parametrize("re,rtmss", [(1e-10, 0.5), (1e-2, 0.0), (1e-6, 0.5)])
def test_thin_branch_rank_at_most_cols(gpu_pkg, re, rtmss):
    """sthosvd.cpp:75-76,91-99: step 3 of a (200, 12, 10) tensor of rank (120, 12, 10)
    unfolds to 200 x 120 (rows > cols): only 120 singular values exist, so the rank
    never exceeds 120, even at a zero budget (rtmss = 0)."""
    rng = np.random.default_rng(3)
    core = rng.standard_normal((120, 12, 10))
    u = [np.linalg.qr(rng.standard_normal((n, r)))[0] for n, r in [(200, 120), (12, 12), (10, 10)]]
    x = np.einsum("abc,ia,jb,kc->ijk", core, *u)
    res = gpu_pkg.compress(gpu_pkg.SourceBuffer.from_array(x), gpu_pkg.Params(target_re=re, rtmss=rtmss))
    ref = oracle.compress(x, target_re=re, rtmss=rtmss)
    assert res.ranks == ref.ranks
    assert res.ranks[0] <= 120
    assert abs(len(res.container) - len(ref.container)) <= 0.01 * len(ref.container)


@pytest.mark.parametrize("backend,shape", [(0, (12, 30, 400)), (2, (6, 10, 90))])
def test_thin_branch_subspaces(gpu_pkg, backend, shape):
    x = synth.small("blobs", shape, seed=4)  # processing order (0, 1, 2): the last step has rows > cols
    tgt = 1e-6 * float((x ** 2).sum())
    a = gpu_pkg.sthosvd(x, tgt, backend=backend)
    b = oracle.sthosvd(x, tgt, backend=backend)
    assert a["ranks"] == b["ranks"]
    for mode, (fa, fb) in enumerate(zip(a["factors"], b["factors"])):
        assert fa.shape == fb.shape
        assert principal_sine(fa, fb) <= subspace_tol(b["sigma2"][mode], b["ranks"][mode])


# ---------------------------------------------------------------- rank tie band
def _orthogonal_rank(sig, dims, seed=0):
    rng = np.random.default_rng(seed)
    R = len(sig)
    us = [np.linalg.qr(rng.standard_normal((n, R)))[0] for n in dims]
    return np.einsum("k,ik,jk,lk->ijl", sig, *us)


def test_rank_tie_band_reported(gpu_pkg):
    """A budget placed exactly on a cutoff's tail sum is flagged (mode 0: its
    Gram eigenvalues are sig^2 exactly, the budget is rtmss * target / d)."""
    sig = 2.0 ** -np.arange(12, dtype=np.float64)
    x = _orthogonal_rank(sig, (32, 36, 40))  # mode 0 is processed first
    tail5 = float((sig[5:] ** 2).sum())
    res = gpu_pkg.compress(gpu_pkg.SourceBuffer.from_array(x), gpu_pkg.Params(target_sse=3.0 / 0.5 * tail5))
    assert res.rank_tie_modes & 1
    res2 = gpu_pkg.compress(gpu_pkg.SourceBuffer.from_array(x), gpu_pkg.Params(target_sse=3.0 / 0.5 * 1.5 * tail5))
    assert not (res2.rank_tie_modes & 1)


@pytest.mark.parametrize("n0", [1300, 1700])
def test_mode_above_1024_against_oracle(gpu_pkg, n0):
    """A mode of more than 1024 rows processed first (Gram route, full
    eigensolver at n0, the factor codec's reflectors and expansion on n0-row
    columns): ranks, container size and RE against the oracle, and the
    device decompress of the container."""
    rng = np.random.default_rng(n0)
    shape, terms = (n0, 40, 36), 32
    w = 0.82 ** np.arange(terms)
    u = [np.linalg.qr(rng.standard_normal((m, terms)))[0] for m in shape]
    x = np.einsum("t,it,jt,kt->ijk", w, *u) + 1e-7 * rng.standard_normal(shape)
    prm = dict(target_re=1e-3)
    res = gpu_pkg.compress(gpu_pkg.SourceBuffer.from_array(x), gpu_pkg.Params(mode_order=[0, 1, 2], **prm))
    ref = oracle.compress(x, mode_order=[0, 1, 2], **prm)
    assert res.ranks == ref.ranks, (res.ranks, ref.ranks)
    assert abs(len(res.container) - len(ref.container)) <= 0.01 * len(ref.container)
    e = rel_err(oracle.decompress(res.container, x.shape), x)
    er = rel_err(oracle.decompress(ref.container, x.shape), x)
    assert abs(e - er) <= 0.01 * er, (e, er)
    y = gpu_pkg.decompress_tensor(res.container)
    assert abs(rel_err(np.asarray(y, np.float64).reshape(x.shape), x) - e) <= 1e-3 * e


def test_eigensolver_size_limit_message(gpu_pkg):
    g = np.eye(2400)
    with pytest.raises(gpu_pkg.TucompError, match="supports mode sizes up to"):
        gpu_pkg.eig(g, 1)


def test_early_full_planes_same_container(gpu_pkg, monkeypatch):
    """Large cores code the full planes above the breakpoint beside the plan
    (speculative sign fold) and append the last plane at finalisation; the
    container must be byte-identical to coding every plane at once."""
    x = config_input("c2")
    src = gpu_pkg.SourceBuffer.from_array(x)
    a = gpu_pkg.compress(src, gpu_pkg.Params(target_re=1e-6))
    assert int(np.prod(a.ranks)) > (1 << 20)
    monkeypatch.setenv("TCB_EARLY_PLANES", "1")
    b = gpu_pkg.compress(src, gpu_pkg.Params(target_re=1e-6))
    assert a.container == b.container
