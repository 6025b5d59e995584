"""The sharded mode loop (shard.py) on the device kernels: at world size 1 it
must reproduce pipeline::compress byte for byte (same kernels, same order)."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,shape,re", [("sin_decay", (48, 40, 36), 1e-4), ("sin", (32, 32, 32), 1e-3)])
def test_sharded_world1_matches_compress(gpu_pkg, kind, shape, re):
    import torch

    from paper_2107_01384_b200 import shard

    x = synth.small(kind, shape, seed=5)
    ref = gpu_pkg.compress(gpu_pkg.SourceBuffer.from_array(x), gpu_pkg.Params(target_re=re))
    xt = torch.from_numpy(x).cuda()
    got = shard.compress_sharded(xt, list(shape), gpu_pkg.Dtype.float64, gpu_pkg.Params(target_re=re))
    assert got.ranks == ref.ranks
    assert got.container == ref.container


def test_sharded_per_stage_path_world1_matches_compress(gpu_pkg, monkeypatch):
    """The per-stage Python mode loop (DeviceOps) is the fallback for unequal
    slabs and off-Gram steps: it too must reproduce compress byte for byte
    (compress with its separate norm pass, which the per-stage path also takes;
    the default reads |A|^2 off the first Gram, a different rounding)."""
    import torch

    monkeypatch.setenv("TCB_NORM_PASS", "1")
    from paper_2107_01384_b200 import shard

    x = synth.small("sin_decay", (40, 36, 30), seed=9)
    prm = gpu_pkg.Params(target_re=1e-4)
    ref = gpu_pkg.compress(gpu_pkg.SourceBuffer.from_array(x), prm)
    got = shard.compress_sharded(torch.from_numpy(x).cuda(), list(x.shape), gpu_pkg.Dtype.float64, prm,
                                 ops=shard.DeviceOps())
    assert got.ranks == ref.ranks
    assert got.container == ref.container


@pytest.mark.parametrize("order", [[2, 0, 1], [1, 2, 0]])
@pytest.mark.parametrize("f32", [False, True])
def test_sharded_library_path_orders_and_dtypes(gpu_pkg, order, f32):
    """The library's sharded pipeline (tcb_compress_sharded_device) with a
    non-identity processing order and a float32 source equals compress."""
    import torch

    from paper_2107_01384_b200 import shard

    x = synth.small("sin_decay", (36, 28, 44), seed=3)
    dt = gpu_pkg.Dtype.float32 if f32 else gpu_pkg.Dtype.float64
    xs = x.astype(np.float32) if f32 else x
    prm = gpu_pkg.Params(target_re=1e-3, mode_order=order)
    ref = gpu_pkg.compress(gpu_pkg.SourceBuffer.from_array(xs), prm)
    got = shard._compress_sharded_cpp(torch.from_numpy(xs).cuda(), list(x.shape), dt, prm, None, 1, 0)
    assert got.ranks == ref.ranks
    assert got.container == ref.container


def test_sharded_library_rejects_wrong_slab(gpu_pkg):
    import torch

    from paper_2107_01384_b200 import TucompError, shard

    x = synth.small("sin", (16, 16, 16), seed=1)
    with pytest.raises(TucompError, match="ingest: buffer holds"):
        shard._compress_sharded_cpp(torch.from_numpy(x[:, :, :8].copy()).cuda(), [16, 16, 16],
                                    gpu_pkg.Dtype.float64, gpu_pkg.Params(target_re=1e-3), None, 1, 0)
