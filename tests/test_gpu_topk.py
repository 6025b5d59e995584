"""Certified top-p eigensolver (csrc/topk.cu) against the full tridiagonal
solver (forced with TCB_NO_TOPK=1): same ranks, discarded energy and factor
subspaces, and the same containers within the parity tolerances."""
import os

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu


def _factor(torch, gram, budget, full):
    from paper_2107_01384_b200 import shard

    old = os.environ.get("TCB_NO_TOPK")
    os.environ["TCB_NO_TOPK"] = "1" if full else "0"
    try:
        u, r, disc = shard.DeviceOps().factor_from_gram(torch.from_numpy(gram).cuda(), budget)
    finally:
        if old is None:
            del os.environ["TCB_NO_TOPK"]
        else:
            os.environ["TCB_NO_TOPK"] = old
    return u.cpu().numpy(), r, disc


def _sine(a, b):
    """largest principal-angle sine between the column spans of a and b"""
    qa, _ = np.linalg.qr(a)
    qb, _ = np.linalg.qr(b)
    return np.linalg.norm(qb - qa @ (qa.T @ qb), 2)


@pytest.mark.parametrize("n,rank,decay,noise", [(256, 12, 1.0, 1e-10), (200, 20, 0.5, 1e-8), (128, 5, 3.0, 0.0),
                                                (300, 24, 0.2, 1e-12)])
def test_topk_matches_full_solver(gpu_pkg, n, rank, decay, noise):
    import torch

    rng = np.random.default_rng(n + rank)
    a = rng.standard_normal((n, rank)) * np.exp(-decay * np.arange(rank))[None, :]
    g = a @ a.T + noise * np.eye(n)
    g = 0.5 * (g + g.T)
    ev = np.linalg.eigvalsh(g)[::-1]
    budget = 0.5 * ev[rank - 2:].sum()  # cutoff a couple of vectors inside the signal rank
    u_f, r_f, d_f = _factor(torch, g, budget, full=False)
    u_s, r_s, d_s = _factor(torch, g, budget, full=True)
    assert r_f == r_s
    assert abs(d_f - d_s) <= 1e-9 * ev[0] + 1e-6 * abs(d_s)
    assert _sine(u_f, u_s) < 1e-6  # the parity bar; both solvers sit near eps |G| / gap
    # the same sign convention (largest |u| positive, first on ties) up to roundoff
    assert np.allclose(u_f, u_s, atol=1e-6)


@pytest.mark.parametrize("kind,shape,re", [("sin_decay", (256, 96, 80), 1e-4), ("blobs", (160, 128, 100), 1e-3),
                                           ("sin", (200, 120, 64), 1e-2)])
def test_topk_end_to_end(gpu_pkg, kind, shape, re):
    x = synth.small(kind, shape, seed=3)
    src = gpu_pkg.SourceBuffer.from_array(x)
    old = os.environ.get("TCB_NO_TOPK")
    try:
        os.environ["TCB_NO_TOPK"] = "0"
        fast = gpu_pkg.compress(src, gpu_pkg.Params(target_re=re))
        os.environ["TCB_NO_TOPK"] = "1"
        full = gpu_pkg.compress(src, gpu_pkg.Params(target_re=re))
    finally:
        if old is None:
            os.environ.pop("TCB_NO_TOPK", None)
        else:
            os.environ["TCB_NO_TOPK"] = old
    assert fast.ranks == full.ranks
    assert abs(len(fast.container) - len(full.container)) <= 0.01 * len(full.container)
    rel = [np.linalg.norm(oracle.decompress(r.container, shape) - x) / np.linalg.norm(x) for r in (fast, full)]
    assert max(rel) <= 1.05 * re  # the hybrid error model's slack, as in the oracle parity tests
    assert abs(rel[0] - rel[1]) <= 0.01 * rel[1]
    # and both against the CPU oracle, not only each other
    ref = oracle.compress(x, target_re=re)
    assert fast.ranks == ref.ranks, (fast.ranks, ref.ranks)
    assert abs(len(fast.container) - len(ref.container)) <= 0.01 * len(ref.container)
    rel_ref = np.linalg.norm(oracle.decompress(ref.container, shape) - x) / np.linalg.norm(x)
    assert abs(rel[0] - rel_ref) <= 0.01 * rel_ref
