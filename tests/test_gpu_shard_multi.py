"""The library's sharded pipeline at world sizes 2 and 3 on one GPU (SURVEY
8(e)): ranks are separate processes sharing the device; the collectives run
through tcb_host_collectives over torch.distributed gloo, so no rank's kernel
ever waits on another rank's.

* encode only: every rank holds the same Tucker factorization and codes its
  share of the core's blocks (exchanging exact block statistics, the crossing
  scan and the split probe, then gathering payloads) -- rank 0's container is
  byte-identical to the unsharded encoder's;
* full compress: the slabs of the last processed mode are sharded (partial
  Grams all-reduced, shard-local TTM, shard-local encoding) -- against the
  single-process compress and the oracle within the parity tolerances."""
import os
import pickle
import tempfile

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu


def _worker(rank, world, initf, outdir, mode):
    import torch
    import torch.distributed as dist

    import paper_2107_01384_b200 as tcb
    from paper_2107_01384_b200 import shard

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"file://{initf}", rank=rank, world_size=world)
    x = synth.small("sin_decay", (64, 60, 72), seed=11)
    params = tcb.Params(target_re=1e-5)
    if mode == "encode":
        tgt = float((x ** 2).sum()) * 1e-10
        st = tcb.sthosvd(x, 0.5 * tgt)
        dev = torch.device("cuda", 0)
        order = st["order"]
        core = torch.from_numpy(np.ascontiguousarray(st["core"])).to(dev)
        facs = [torch.from_numpy(np.ascontiguousarray(f)).to(dev) for f in st["factors"]]
        res = shard.encode_tucker_sharded(core, facs, list(x.shape), st["ranks"], order, st["trunc"],
                                          tcb.Dtype.float64, float((x ** 2).sum()), tgt, tcb.Params(target_sse=tgt))
    else:
        lo, hi = shard.shard_bounds(x.shape[2], world, rank)
        xs = torch.from_numpy(np.ascontiguousarray(x[:, :, lo:hi])).cuda()
        res = shard.compress_sharded_host(xs, list(x.shape), tcb.Dtype.float64, params)
    if rank == 0:
        with open(os.path.join(outdir, "out.pkl"), "wb") as f:
            pickle.dump({"container": res.container, "ranks": res.ranks}, f)
    dist.barrier()
    dist.destroy_process_group()


def _run(world, mode):
    import torch.multiprocessing as mp

    with tempfile.TemporaryDirectory() as td:
        initf = os.path.join(td, "init")
        mp.start_processes(_worker, args=(world, initf, td, mode), nprocs=world, join=True, start_method="spawn")
        with open(os.path.join(td, "out.pkl"), "rb") as f:
            return pickle.load(f)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_encode_bitwise_equals_unsharded(gpu_pkg, world):
    x = synth.small("sin_decay", (64, 60, 72), seed=11)
    tgt = float((x ** 2).sum()) * 1e-10
    st = gpu_pkg.sthosvd(x, 0.5 * tgt)
    assert int(np.prod(st["ranks"])) > 4096 * world  # several blocks per rank
    out = _run(world, "encode")
    import torch

    from paper_2107_01384_b200 import shard

    dev = torch.device("cuda", 0)
    core = torch.from_numpy(np.ascontiguousarray(st["core"])).to(dev)
    facs = [torch.from_numpy(np.ascontiguousarray(f)).to(dev) for f in st["factors"]]
    ref = shard.DeviceOps().encode(core, facs, list(x.shape), st["ranks"], st["order"], st["trunc"],
                                   gpu_pkg.Dtype.float64, float((x ** 2).sum()), tgt,
                                   gpu_pkg.Params(target_sse=tgt))
    assert out["container"] == ref.container


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_compress_matches_oracle(gpu_pkg, world):
    x = synth.small("sin_decay", (64, 60, 72), seed=11)
    out = _run(world, "compress")
    ref = oracle.compress(x, target_re=1e-5)
    assert out["ranks"] == ref.ranks
    assert abs(len(out["container"]) - len(ref.container)) <= 0.01 * len(ref.container)
    y = oracle.decompress(out["container"], x.shape)
    yr = oracle.decompress(ref.container, x.shape)
    e = np.linalg.norm(y - x) / np.linalg.norm(x)
    er = np.linalg.norm(yr - x) / np.linalg.norm(x)
    assert abs(e - er) <= 0.01 * er
