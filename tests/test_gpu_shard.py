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
