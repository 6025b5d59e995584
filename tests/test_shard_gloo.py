"""Multi-rank ST-HOSVD orchestration (paper_2107_01384_b200/shard.py) on CPU:
world_size 2 and 3 over gloo, per-rank compute by a numpy stand-in for the
device kernels (the eigensolver is the oracle's SelfAdjointEigenSolver
restatement), checked against the single-rank run of the same code and
against the oracle's unsharded sthosvd."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth


class NumpyOps:
    def sumsq(self, x):
        return float((x.double() ** 2).sum()), bool(torch.isfinite(x).all())

    def permute(self, x, perm):
        return x.permute(*perm).contiguous()

    def gram(self, b2):
        return b2 @ b2.T

    def _rank_and_u(self, s2, vecs, budget):
        r, disc = oracle.pick_rank(s2, budget)
        if r == 0:
            r, disc = 1, disc - s2[0]
        u = vecs[:, :r].copy()
        for j in range(r):
            i = int(np.argmax(np.abs(u[:, j])))
            if u[i, j] < 0:
                u[:, j] = -u[:, j]
        return torch.from_numpy(u), r, disc

    def factor_from_gram(self, g, budget):
        ev, vec = oracle.eig(g.numpy())
        ev, vec = ev[::-1], vec[:, ::-1]
        return self._rank_and_u(np.maximum(0.0, ev), vec, budget)

    def ttm(self, b2, u):
        return b2.T @ u

    def mode_step(self, b2, budget, backend):
        rows, cols = b2.shape
        if backend == 1 or (backend == 0 and rows <= cols):
            u, r, disc = self.factor_from_gram(self.gram(b2), budget)
        else:
            uu, sv, _ = np.linalg.svd(b2.numpy(), full_matrices=False)
            u, r, disc = self._rank_and_u(sv.astype(np.float64) ** 2, uu, budget)
        return u, self.ttm(b2, u), r, disc


def _worker(rank, world, port, shape, target, order, path):
    os.environ.setdefault("GLOO_SOCKET_IFNAME", "lo")
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    from paper_2107_01384_b200 import shard

    x = synth.small("sin_decay", shape, seed=11)
    p = list(order) if order is not None else shard.stable_ascending(shape)
    ax = p[-1]
    lo, hi = shard.shard_bounds(shape[ax], world, rank)
    xl = torch.from_numpy(np.ascontiguousarray(np.take(x, np.arange(lo, hi), axis=ax)))
    f = shard.sthosvd_sharded(xl, list(shape), target, NumpyOps(), order=order)
    if rank == 0:
        np.savez(path, core=f.core.numpy(), ranks=np.array(f.ranks), trunc=np.array(f.trunc), order=np.array(f.order),
                 norm=f.norm_sq, **{f"f{i}": f.factors[i].numpy() for i in range(len(shape))})
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world, shape, target, order=None):
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "out.npz")
        mp.spawn(_worker, args=(world, _free_port(), shape, target, order, path), nprocs=world, join=True)
        return dict(np.load(path))


@pytest.mark.parametrize("shape,frac,order", [((12, 14, 9), 1e-4, None), ((10, 7, 13), 1e-2, None),
                                              ((10, 4, 6), 0.3, (1, 0, 2))])
def test_sharded_matches_single_rank_and_oracle(shape, frac, order):
    x = synth.small("sin_decay", shape, seed=11)
    target = frac * float((x ** 2).sum())
    one = _run(1, shape, target, order)
    ref = oracle.sthosvd(x, target, order=order)
    assert one["ranks"].tolist() == ref["ranks"]
    for world in (2, 3):
        got = _run(world, shape, target, order)
        assert got["ranks"].tolist() == one["ranks"].tolist()
        assert np.allclose(got["trunc"], one["trunc"], rtol=1e-9, atol=1e-12 * target)
        assert abs(got["norm"] - one["norm"]) <= 1e-12 * one["norm"]
        for i in range(len(shape)):
            assert np.allclose(got[f"f{i}"], one[f"f{i}"], atol=1e-9)
        assert np.allclose(got["core"], one["core"], atol=1e-9 * np.abs(one["core"]).max())
        # and the unsharded oracle
        for i in range(len(shape)):
            assert np.allclose(got[f"f{i}"], ref["factors"][i], atol=1e-8)
