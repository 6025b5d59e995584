"""The Ozaki-scheme Gram and TTM on the INT8 tensor cores (csrc/ozaki.cu)
against fp64 references: five 7-bit digit slices per row / column truncate
each value 34 bits below its row's (column's) largest and the dropped digit
levels weigh <= 2^-35 per term, so every entry is within 2^-32 (Gram) / 2^-30
(TTM, 2.8e-10 measured) of |x_i| |x_j| from the exact product sum, the Gram is bitwise
symmetric with the fp64 row sums of squares on its diagonal, and the result
is deterministic.  The tcgen05 kernel (csrc/ozmma.cu) and the cuBLASLt IMMA
path (TCB_OZAKI_LT=1) compute the same integers, so they agree bit for bit.
End to end, a compress whose mode loop takes the INT8 path matches the oracle
within the parity bar."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _data(rows, cols, kind, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(rows, cols, dtype=torch.float64, device="cuda", generator=g)
    if kind == "range":  # rows and columns over many binades, some exact zeros
        x *= torch.exp2(torch.randint(-20, 20, (rows, 1), device="cuda", generator=g).double())
        x *= torch.exp2(torch.randint(-8, 8, (1, cols), device="cuda", generator=g).double())
        x[:, ::7] = 0.0
    elif kind == "f32":  # an fp32 source cast to double, as c5's mode 0
        x = x.float().double()
    return x


@pytest.mark.parametrize("rows,cols,kind", [(64, 5000, "normal"), (300, 70001, "range"), (1024, 40000, "f32"),
                                            (17, 33, "normal"), (256, 1 << 18, "normal")])
def test_gram_ozaki_against_fp64(gpu_pkg, rows, cols, kind):
    from paper_2107_01384_b200 import shard

    ops = shard.DeviceOps()
    x = _data(rows, cols, kind, 1)
    g = ops.gram_ozaki(x)
    ref = x @ x.t()
    nrm = x.norm(dim=1)
    bound = torch.outer(nrm, nrm) * 2.0 ** -32 + 1e-300
    assert bool(((g - ref).abs() <= bound).all())
    assert torch.equal(g, g.t())  # bitwise symmetric (exact integer levels)
    assert torch.allclose(torch.diagonal(g), (x * x).sum(dim=1), rtol=1e-13, atol=0)
    assert torch.equal(g, ops.gram_ozaki(x))  # deterministic


@pytest.mark.parametrize("rows,cols,r,kind", [(200, 30000, 70, "normal"), (1024, 50000, 650, "f32"),
                                              (300, 4097, 5, "range"), (33, 100, 33, "normal")])
def test_ttm_ozaki_against_fp64(gpu_pkg, rows, cols, r, kind):
    from paper_2107_01384_b200 import shard

    ops = shard.DeviceOps()
    b = _data(rows, cols, kind, 2)
    u = torch.linalg.qr(torch.randn(rows, r, dtype=torch.float64, device="cuda"))[0]
    out = ops.ttm_ozaki(b, u)
    ref = b.t() @ u
    bound = torch.outer(b.norm(dim=0), u.norm(dim=0)) * 2.0 ** -30 + 1e-300
    assert bool(((out - ref).abs() <= bound).all())
    assert torch.equal(out, ops.ttm_ozaki(b, u))


@pytest.mark.parametrize("rows,cols", [(1024, 1 << 18), (300, 70001), (129, 40000), (97, 33000), (17, 33)])
def test_gram_tcgen05_equals_cublaslt(gpu_pkg, monkeypatch, rows, cols):
    """Partial 128 x 96 tiles, several 2^15 k-chunks, the c5 mode-0 width."""
    from paper_2107_01384_b200 import shard

    ops = shard.DeviceOps()
    x = _data(rows, cols, "range", 3)
    g_tc = ops.gram_ozaki(x)
    monkeypatch.setenv("TCB_OZAKI_LT", "1")
    g_lt = ops.gram_ozaki(x)
    assert torch.equal(g_tc, g_lt)


@pytest.mark.parametrize("rows,cols,r", [(1024, 50000, 650), (300, 4097, 5), (33, 100, 33), (200, 30001, 97),
                                         (1000, 2000, 96)])
def test_ttm_tcgen05_equals_cublaslt(gpu_pkg, monkeypatch, rows, cols, r):
    from paper_2107_01384_b200 import shard

    ops = shard.DeviceOps()
    b = _data(rows, cols, "range", 4)
    u = torch.linalg.qr(torch.randn(rows, r, dtype=torch.float64, device="cuda"))[0]
    o_tc = ops.ttm_ozaki(b, u)
    monkeypatch.setenv("TCB_OZAKI_LT", "1")
    o_lt = ops.ttm_ozaki(b, u)
    assert torch.equal(o_tc, o_lt)


def test_compress_int8_path_matches_oracle(gpu_pkg):
    """A 256 x 512 x 512 fp32 random field: the first mode's unfolding has 2^18
    columns, so the mode loop starts on the INT8 path; ranks equal, container
    and RE within 1 % of the oracle's."""
    import oracle
    import synth

    x = synth.grf_torch(n=512, kmax=170, seed=3)[:256].contiguous()
    xh = x.cpu().numpy()
    src = gpu_pkg.SourceBuffer.from_array(xh)
    p = gpu_pkg.Params(target_re=1e-2)
    a = gpu_pkg.compress(src, p)
    ref = oracle.compress(xh, target_re=1e-2)
    assert a.ranks == ref.ranks
    assert abs(len(a.container) - len(ref.container)) <= 0.01 * len(ref.container)
    ya = oracle.decompress(a.container, xh.shape)
    yr = oracle.decompress(ref.container, xh.shape)
    xd = xh.astype(np.float64)
    ea = np.linalg.norm(ya - xd) / np.linalg.norm(xd)
    er = np.linalg.norm(yr - xd) / np.linalg.norm(xd)
    assert abs(ea - er) <= 0.01 * er
