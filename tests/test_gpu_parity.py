"""GPU parity tests: every device kernel of the compress path against the CPU
oracle (bit-exact for integer/bitstream work, stated tolerances for FP)."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def principal_sine(u, v):
    """largest principal-angle sine between span(u) and span(v) (orthonormal
    columns): ||(I - V V^T) U||_2, accurate for small angles (unlike sqrt(1-cos^2))."""
    return float(np.linalg.norm(u - v @ (v.T @ u), 2))


# ---------------------------------------------------------------- dense kernels
@pytest.mark.parametrize("rows,cols", [(64, 4096), (100, 2500), (256, 65536), (37, 1001), (5, 7)])
def test_gram_matches_fp64_reference(gpu_pkg, rows, cols):
    b = np.random.default_rng(rows + cols).standard_normal((rows, cols))
    g = gpu_pkg.gram(b)
    ref = b @ b.T
    # tolerance: fp64 accumulation over `cols` terms
    assert np.abs(g - ref).max() <= 1e-13 * cols * np.abs(ref).max() ** 0 * np.abs(b).max() ** 2 * 10
    assert np.array_equal(g, g.T)


@pytest.mark.parametrize("rows,cols,r", [(64, 4096, 20), (256, 65536, 64), (100, 2500, 100), (7, 33, 3),
                                         (256, 1001, 255)])
def test_ttm_matches_fp64_reference(gpu_pkg, rows, cols, r):
    rng = np.random.default_rng(rows * 7 + r)
    b = rng.standard_normal((rows, cols))
    u = rng.standard_normal((rows, r))
    out = gpu_pkg.ttm(b, u)
    ref = b.T @ u
    assert np.abs(out - ref).max() <= 1e-12 * rows * np.abs(ref).max()


def test_gram_is_deterministic(gpu_pkg):
    b = np.random.default_rng(0).standard_normal((256, 8192))
    assert np.array_equal(gpu_pkg.gram(b), gpu_pkg.gram(b))


@pytest.mark.parametrize("n", [1, 2, 3, 17, 64, 100, 256, 500, 601, 700, 1024, 1500, 2048])
def test_eigensolver_matches_lapack(gpu_pkg, n):
    rng = np.random.default_rng(n)
    b = rng.standard_normal((n, 3 * n + 5))
    # graded spectrum like a Tucker unfolding Gram
    b *= (np.arange(1, n + 1) ** -1.5)[:, None]
    g = b @ b.T
    w_ref, v_ref = np.linalg.eigh(g)
    w_ref, v_ref = w_ref[::-1], v_ref[:, ::-1]
    r = max(1, n // 3)
    ev, u = gpu_pkg.eig(g, r)
    assert np.abs(ev - w_ref).max() <= 1e-12 * abs(w_ref).max() * max(1, n) ** 0.5
    assert np.abs(u.T @ u - np.eye(r)).max() <= 1e-12
    assert principal_sine(u, v_ref[:, :r]) <= 1e-6
    # sign convention: the largest-magnitude entry of every column is non-negative
    for j in range(r):
        assert u[np.argmax(np.abs(u[:, j])), j] >= 0


def test_eigensolver_clusters_stay_orthonormal(gpu_pkg):
    n = 128
    q, _ = np.linalg.qr(np.random.default_rng(1).standard_normal((n, n)))
    w = np.concatenate([np.linspace(10, 5, 8), 1e-6 * (1 + 1e-9 * np.arange(n - 8))])
    g = (q * w) @ q.T
    g = 0.5 * (g + g.T)
    ev, u = gpu_pkg.eig(g, n)
    assert np.abs(u.T @ u - np.eye(n)).max() <= 1e-10
    assert principal_sine(u[:, :8], q[:, :8]) <= 1e-8


# ---------------------------------------------------------------- quantisation
@pytest.mark.parametrize("shape", [(8, 9, 10), (59, 58, 57), (3, 1, 4), (1, 1, 1)])
def test_quantize_bit_exact(gpu_pkg, shape):
    core = synth.small("random", shape, seed=sum(shape)) * np.logspace(0, -8, int(np.prod(shape))).reshape(shape)
    a = gpu_pkg.quantize(core)
    b = oracle.quantize(core)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2] and a[3] == b[3]
    for x, y in zip(a[4], b[4]):
        assert np.array_equal(x, y)  # serial-order slice norms: bitwise


def test_quantize_zero_core(gpu_pkg):
    mag, neg, k, zero, sn = gpu_pkg.quantize(np.zeros((4, 3, 2)))
    assert zero and k == 0


def test_quantize_spec_example(gpu_pkg):
    mag, neg, k, zero, _ = gpu_pkg.quantize(np.array([[[0.5, -0.25]]]))
    assert k == 64 and mag.tolist() == [2 ** 63, 2 ** 62] and neg.tolist() == [0, 1]


# ---------------------------------------------------------------- encoder
def _core_mags(shape=(40, 41, 42), seed=0, decay=6.0):
    rng = np.random.default_rng(seed)
    idx = np.indices(shape).sum(0).astype(np.float64)
    core = rng.standard_normal(shape) * np.exp(-decay * idx / idx.max())
    mag, neg, k, zero, sn = oracle.quantize(core)
    return mag, neg


@pytest.mark.parametrize("frac", [1e-1, 1e-3, 1e-6, 1e-9, 1e-12, 0.0, 2.0])
@pytest.mark.parametrize("split", [True, False])
@pytest.mark.parametrize("coder", [0, 1])
def test_encoder_bitstream_bit_exact(gpu_pkg, frac, split, coder):
    mag, neg = _core_mags()
    tot = float((mag.astype(np.float64) ** 2).sum())
    tgt = tot * frac
    s_gpu, lp_gpu, ach_gpu, dec_gpu, _ = gpu_pkg.encode(mag, neg, tgt, coder=coder, split=split)
    s_ref, lp_ref, ach_ref, dec_ref = oracle.encode(mag, neg, tgt, coder=coder, split=split)
    assert lp_gpu == lp_ref
    assert np.array_equal(dec_gpu, dec_ref)
    assert s_gpu == s_ref
    assert ach_gpu == pytest.approx(ach_ref, rel=1e-12, abs=0)


@pytest.mark.parametrize("frac", [1e-3, 1e-6])
@pytest.mark.parametrize("split", [True, False])
def test_encoder_bitstream_bit_exact_large(gpu_pkg, frac, split):
    """A 2.2M-coefficient core (above 2^20): the sampled breakpoint estimate, the
    table-driven exact plane statistics, the speculative split probe and the
    densest planes coded on their own stream all take part; the stream is the
    oracle's byte for byte."""
    mag, neg = _core_mags(shape=(130, 130, 131), seed=4, decay=9.0)
    tot = float((mag.astype(np.float64) ** 2).sum())
    tgt = tot * frac
    s_gpu, lp_gpu, ach_gpu, dec_gpu, _ = gpu_pkg.encode(mag, neg, tgt, coder=0, split=split)
    s_ref, lp_ref, ach_ref, dec_ref = oracle.encode(mag, neg, tgt, coder=0, split=split)
    assert lp_gpu == lp_ref
    assert np.array_equal(dec_gpu, dec_ref)
    assert s_gpu == s_ref
    assert ach_gpu == pytest.approx(ach_ref, rel=1e-12, abs=0)


@pytest.mark.parametrize("fixed", [63, 50, 40, 10, 0])
def test_encoder_fixed_plane_bit_exact(gpu_pkg, fixed):
    mag, neg = _core_mags((17, 19, 23), seed=5)
    a = gpu_pkg.encode(mag, neg, 0.0, split=False, fixed_plane=fixed)
    b = oracle.encode(mag, neg, 0.0, split=False, fixed_plane=fixed)
    assert a[0] == b[0] and a[1] == b[1] and np.array_equal(a[3], b[3])


@pytest.mark.parametrize("block", [4096, 5000, 100000])
def test_encoder_block_sizes(gpu_pkg, block):
    mag, neg = _core_mags((50, 60, 70), seed=9)
    tot = float((mag.astype(np.float64) ** 2).sum())
    a = gpu_pkg.encode(mag, neg, tot * 1e-7, block_size=block)
    b = oracle.encode(mag, neg, tot * 1e-7, block_size=block)
    assert a[0] == b[0] and a[1] == b[1]


def test_encoder_edge_cases(gpu_pkg):
    for mag in [np.zeros(0, np.uint64), np.zeros(10, np.uint64), np.array([1], np.uint64),
                np.array([2 ** 63, 0, 1, 2 ** 64 - 1], np.uint64)]:
        neg = (np.arange(mag.size) % 2).astype(np.uint8)
        for tgt in [0.0, 1.0, 1e300]:
            a = gpu_pkg.encode(mag, neg, tgt)
            b = oracle.encode(mag, neg, tgt)
            assert a[0] == b[0] and a[1] == b[1], (mag, tgt)


@pytest.mark.parametrize("seed", range(4))
def test_encode_symbols_bit_exact(gpu_pkg, seed):
    rng = np.random.default_rng(seed)
    syms = np.concatenate([rng.geometric(0.05, 3000) - 1, rng.integers(0, 2 ** 32 - 1, 50)]).astype(np.uint64)
    rng.shuffle(syms)
    for coder in (0, 1):
        assert gpu_pkg.encode_symbols(coder, syms) == oracle.encode_symbols(coder, syms)
        assert gpu_pkg.encode_symbols(coder, []) == oracle.encode_symbols(coder, [])


@pytest.mark.parametrize("kind", ["constant", "distinct", "long", "runs", "huge", "skewed"])
def test_encode_symbols_model_edges(gpu_pkg, kind):
    """Chunked adaptive model: repeats inside a chunk, > 2048 distinct symbols
    (shared-memory model overflow -> global-scratch rerun), many halvings."""
    rng = np.random.default_rng(7)
    if kind == "constant":
        syms = np.zeros(5000, np.uint64)
    elif kind == "distinct":
        syms = rng.permutation(np.arange(6000, dtype=np.uint64) * 2654435761 % (2 ** 32))
    elif kind == "long":
        syms = (rng.geometric(0.2, 40000) - 1).astype(np.uint64)
    elif kind == "huge":  # thousands of output chunks, hundreds of halvings, carries across chunks
        syms = (rng.geometric(0.02, 1_500_000) - 1).astype(np.uint64)
    elif kind == "skewed":  # near-certain symbols: long 0xFF runs in the output, rare escapes
        syms = np.where(rng.random(300_000) < 0.999, 0, rng.integers(1, 3000, 300_000)).astype(np.uint64)
    else:
        syms = np.repeat(rng.integers(0, 40, 700), rng.integers(1, 60, 700)).astype(np.uint64)
    assert gpu_pkg.encode_symbols(0, syms) == oracle.encode_symbols(0, syms)


# ---------------------------------------------------------------- factor codec
@pytest.mark.parametrize("n,r", [(40, 10), (64, 59), (30, 30), (1, 1), (100, 3)])
def test_factor_stream_matches_oracle(gpu_pkg, n, r):
    rng = np.random.default_rng(n * 100 + r)
    q, _ = np.linalg.qr(rng.standard_normal((n, r)))
    sn = np.sort(rng.uniform(0.1, 10, r))[::-1]
    dead = np.zeros(r, np.uint8)
    if r > 3:
        dead[-1] = 1
    a = gpu_pkg.encode_factor(q, dead, sn, core_step_log2=-30, term_cap=1e-9)
    b = oracle.encode_factor(q, dead, sn, core_step_log2=-30, term_cap=1e-9)
    assert a["k"] == b["k"] and a["count"] == b["count"] and np.array_equal(a["flips"], b["flips"])
    assert a["plane"] == b["plane"]
    assert a["term"] == pytest.approx(b["term"], rel=1e-6, abs=1e-300)
    assert a["stream"] == b["stream"]


def test_factor_rejects_non_orthonormal(gpu_pkg):
    u = np.ones((5, 2))
    with pytest.raises(gpu_pkg.TucompError, match="not orthonormal"):
        gpu_pkg.encode_factor(u, np.zeros(2, np.uint8), np.ones(2))


# ---------------------------------------------------------------- ST-HOSVD
@pytest.mark.parametrize("kind,shape,frac", [("sin", (32, 32, 32), 1e-6), ("sin_decay", (48, 40, 36), 1e-8),
                                             ("blobs", (20, 50, 50), 1e-4), ("sin", (64, 24, 8), 1e-3),
                                             ("random", (6, 7, 200), 1e-2)])
def test_sthosvd_ranks_and_subspaces(gpu_pkg, kind, shape, frac):
    x = synth.small(kind, shape, seed=1)
    tgt = frac * float((x.astype(np.float64) ** 2).sum())
    a = gpu_pkg.sthosvd(x, tgt)
    b = oracle.sthosvd(x, tgt)
    assert a["ranks"] == b["ranks"] and a["order"] == b["order"]
    for fa, fb in zip(a["factors"], b["factors"]):
        assert principal_sine(fa, fb) <= 1e-6
        assert np.abs(fa.T @ fa - np.eye(fa.shape[1])).max() <= 1e-10
    assert np.allclose(a["trunc"], b["trunc"], rtol=1e-6, atol=1e-9 * tgt)


# ---------------------------------------------------------------- end to end
@pytest.mark.parametrize("kind,shape,dtype,re", [
    ("sin", (64, 64, 64), np.float32, 1e-3),       # c1 (BASELINE configs[0])
    ("sin_decay", (64, 64, 64), np.float64, 1e-4),  # c2 family, reduced
    ("blobs", (25, 60, 60), np.float32, 1e-3),      # c3 family, reduced
    ("sin", (40, 30, 20), np.float64, 1e-2),
])
def test_compress_end_to_end(gpu_pkg, kind, shape, dtype, re):
    x = synth.small(kind, shape, seed=7, dtype=dtype)
    res = gpu_pkg.compress(gpu_pkg.SourceBuffer.from_array(x), gpu_pkg.Params(target_re=re))
    ref = oracle.compress(x, target_re=re)
    assert res.ranks == ref.ranks
    assert abs(len(res.container) - len(ref.container)) <= 0.01 * len(ref.container)
    xd = x.astype(np.float64)
    y = oracle.decompress(res.container, x.shape)
    yr = oracle.decompress(ref.container, x.shape)
    e = np.sqrt(((y - xd) ** 2).sum() / (xd ** 2).sum())
    er = np.sqrt(((yr - xd) ** 2).sum() / (xd ** 2).sum())
    assert abs(e - er) <= 0.01 * er
    assert res.norm_sq == pytest.approx(ref.norm_sq, rel=1e-12)
    assert res.estimate.truncation_sse == pytest.approx(ref.truncation_sse, rel=1e-6)


@pytest.mark.parametrize("gopts,oopts", [
    (dict(coder=1), dict(coder=1)),
    (dict(split_planes=False), dict(split=False)),
    (dict(simple_factor_weights=True), dict(simple=True)),
    (dict(coder=1, split_planes=False, block_size=1024), dict(coder=1, split=False, block_size=1024)),
    (dict(method=1), dict(method=1)),  # zigzag vectorization
    (dict(method=2), dict(method=2)),  # Z-order vectorization
    (dict(method=2, block_size=1024, coder=1), dict(method=2, block_size=1024, coder=1)),
])
def test_compress_coding_options_end_to_end(gpu_pkg, gopts, oopts):
    """Non-default coding options: rANS, non-split planes,
    simple factor weights, small blocks -- against the oracle."""
    x = synth.small("sin_decay", (48, 44, 40), seed=8)
    res = gpu_pkg.compress(gpu_pkg.SourceBuffer.from_array(x), gpu_pkg.Params(target_re=1e-4, **gopts))
    ref = oracle.compress(x, target_re=1e-4, **oopts)
    assert res.ranks == ref.ranks
    assert abs(len(res.container) - len(ref.container)) <= 0.01 * len(ref.container)
    y, yr = oracle.decompress(res.container, x.shape), oracle.decompress(ref.container, x.shape)
    e = np.linalg.norm(y - x) / np.linalg.norm(x)
    er = np.linalg.norm(yr - x) / np.linalg.norm(x)
    assert abs(e - er) <= 0.01 * er
    assert np.max(np.abs(gpu_pkg.decompress_tensor(res.container) - y)) <= 1e-12 * np.max(np.abs(y))


def test_container_parses_with_verbatim_reference_reader(gpu_pkg):
    """The GPU container round-trips byte-for-byte through the reference's own
    read_container/write_container (oracle/_ref, compiled verbatim)."""
    import oracle.ref as R

    if not R.available():
        pytest.skip("oracle/_ref not built")
    x = synth.small("sin", (48, 40, 36), seed=2)
    res = gpu_pkg.compress(gpu_pkg.SourceBuffer.from_array(x), gpu_pkg.Params(target_re=1e-3))
    assert R.container_rewrite(res.container) == res.container
    mag, neg = R.container_core(res.container)
    assert mag.size == int(np.prod(res.ranks))


def test_compress_uint16_permuted_modes(gpu_pkg):
    x = synth.spectral_cube((48, 40, 24), n_materials=4, seed=1)  # c4 family: p != identity
    res = gpu_pkg.compress(gpu_pkg.SourceBuffer.from_array(x), gpu_pkg.Params(target_re=1e-3))
    ref = oracle.compress(x, target_re=1e-3)
    assert res.ranks == ref.ranks
    assert abs(len(res.container) - len(ref.container)) <= 0.01 * len(ref.container)


def test_compress_errors_match_reference(gpu_pkg):
    x = np.ones((4, 4, 4))
    x[1, 1, 1] = np.nan
    with pytest.raises(gpu_pkg.TucompError, match="sthosvd: input contains non-finite values"):
        gpu_pkg.compress(gpu_pkg.SourceBuffer.from_array(x), gpu_pkg.Params(target_re=1e-2))
    y = np.ones((4, 4, 4))
    with pytest.raises(gpu_pkg.TucompError, match="mutually exclusive"):
        gpu_pkg.compress(gpu_pkg.SourceBuffer.from_array(y), gpu_pkg.Params(target_re=1e-2, target_sse=1.0))
    with pytest.raises(gpu_pkg.TucompError, match="no error target"):
        gpu_pkg.compress(gpu_pkg.SourceBuffer.from_array(y), gpu_pkg.Params())
    with pytest.raises(gpu_pkg.TucompError, match="rtmss"):
        gpu_pkg.compress(gpu_pkg.SourceBuffer.from_array(y), gpu_pkg.Params(target_re=1e-2, rtmss=2))
    src = gpu_pkg.SourceBuffer(b"\0" * 10, gpu_pkg.Dtype.float64, [4, 4, 4])
    with pytest.raises(gpu_pkg.TucompError, match="ingest: buffer holds 10 bytes, expected 512"):
        gpu_pkg.compress(src, gpu_pkg.Params(target_re=1e-2))


def test_compress_zero_tensor(gpu_pkg):
    x = np.zeros((8, 8, 8))
    res = gpu_pkg.compress(gpu_pkg.SourceBuffer.from_array(x), gpu_pkg.Params(target_re=1e-2))
    ref = oracle.compress(x, target_re=1e-2)
    assert res.container == ref.container


# ---------------------------------------------------------------- golden vectors (reference's own code)
import hashlib as _hl  # noqa: E402
import json as _json  # noqa: E402
import os as _os  # noqa: E402

_GOLDEN = _json.load(open(_os.path.join(_os.path.dirname(__file__), "golden", "golden.json")))


def _golden_core(g):
    rng = np.random.default_rng(g["seed"])
    shape = tuple(g["shape"])
    idx = np.indices(shape).sum(0).astype(np.float64)
    return rng.standard_normal(shape) * np.exp(-g["decay"] * idx / idx.max())


@pytest.mark.parametrize("g", _GOLDEN["encode"],
                         ids=lambda g: f"c{g['coder']}-s{g['seed']}-f{g['frac']}-sp{int(g['split'])}-fx{g['fixed']}")
def test_gpu_encoder_matches_reference_golden(gpu_pkg, g):
    mag, neg, k, zero, sn = gpu_pkg.quantize(_golden_core(g))
    tot = float((mag.astype(np.float64) ** 2).sum())
    s, lp, ach, dec, _ = gpu_pkg.encode(mag, neg, tot * g["frac"], coder=g["coder"], split=g["split"],
                                        fixed_plane=g["fixed"])
    assert lp == g["last_plane"] and len(s) == g["len"] and _hl.sha256(s).hexdigest() == g["sha"]
    assert _hl.sha256(dec.tobytes()).hexdigest() == g["dec_sha"]


@pytest.mark.parametrize("g", _GOLDEN["quantize"], ids=lambda g: f"seed{g['seed']}")
def test_gpu_quantize_matches_reference_golden(gpu_pkg, g):
    mag, neg, k, zero, sn = gpu_pkg.quantize(_golden_core(g))
    assert k == g["k"] and _hl.sha256(mag.tobytes()).hexdigest() == g["mag_sha"]
    assert [[float(v).hex() for v in ax] for ax in sn] == g["slice_norms_hex"]


@pytest.mark.parametrize("g", _GOLDEN["symbols"], ids=lambda g: f"c{g['coder']}-case{g['case']}")
def test_gpu_entropy_matches_reference_golden(gpu_pkg, g):
    assert gpu_pkg.encode_symbols(g["coder"], g["symbols"]).hex() == g["bytes"]


# ---------------------------------------------------------------- ingest completeness
@pytest.mark.parametrize("dtype", [np.int8, np.uint8, np.int16, np.uint16, np.int32, np.uint32, np.int64, np.uint64,
                                   np.float32, np.float64])
def test_compress_every_source_dtype_with_skip_bytes(gpu_pkg, dtype):
    """container.cpp:51-94: all 10 source dtypes, a skipped prefix, the int64
    precision-loss flag -- ranks, sizes and errors against the oracle."""
    base = synth.small("blobs", (24, 20, 16), seed=11)
    if np.issubdtype(dtype, np.integer):
        info = np.iinfo(dtype)
        hi = min(info.max, 2 ** 62) if dtype in (np.int64, np.uint64) else info.max
        lo = 0 if info.min == 0 else max(info.min, -hi)
        x = np.round((base - base.min()) / np.ptp(base) * (hi - lo) * 0.9 + lo).astype(dtype)
    else:
        x = base.astype(dtype)
    skip = bytes(range(7))
    src = gpu_pkg.SourceBuffer(skip + x.tobytes(), gpu_pkg.Dtype(oracle.DTYPES[np.dtype(dtype)]), x.shape,
                               skip_bytes=len(skip))
    res = gpu_pkg.compress(src, gpu_pkg.Params(target_re=1e-3))
    ref = oracle.compress(x, skip_bytes=skip, target_re=1e-3)
    assert res.ranks == ref.ranks
    assert res.ingest_precision_loss == ref.precision_loss
    assert res.original_bytes == ref.original_bytes == x.nbytes
    assert abs(len(res.container) - len(ref.container)) <= 0.01 * len(ref.container) + 8
    y = oracle.decompress(res.container, x.shape)
    xd = x.astype(np.float64)
    assert np.linalg.norm(y - xd) <= 1.05e-3 * np.linalg.norm(xd)


def test_norm_from_first_gram(gpu_pkg):
    """fp64 inputs take |A|^2 from the first mode's Gram trace (no separate norm
    pass): the reported norm matches numpy, a NaN is still the reference's
    error under either target kind, and a finite input whose squares overflow
    falls back to the norm pass (same outcome as before)."""
    x = synth.small("sin_decay", (40, 36, 28), seed=3)
    res = gpu_pkg.compress(gpu_pkg.SourceBuffer.from_array(x), gpu_pkg.Params(target_re=1e-4))
    assert abs(res.norm_sq - float((x * x).sum())) <= 1e-12 * float((x * x).sum())
    ref = oracle.compress(x, target_re=1e-4)
    assert res.ranks == ref.ranks
    y = x.copy()
    y[3, 4, 5] = np.inf
    for prm in (gpu_pkg.Params(target_re=1e-3), gpu_pkg.Params(target_sse=1.0)):
        with pytest.raises(gpu_pkg.TucompError, match="sthosvd: input contains non-finite values"):
            gpu_pkg.compress(gpu_pkg.SourceBuffer.from_array(y), prm)
    big = x * 1e160  # finite, but the squares overflow: the element scan decides, then
    try:              # the separate-norm path runs (an error there is the old behaviour)
        gpu_pkg.compress(gpu_pkg.SourceBuffer.from_array(big), gpu_pkg.Params(target_sse=1e300))
    except gpu_pkg.TucompError as e:
        assert "non-finite values" not in str(e)


def test_chunked_upload_gram_is_bitwise(gpu_pkg):
    """Pinned fp64 uploads overlap the first Gram with the transfer (column
    chunks, the same split-K plan): the container equals the device-resident
    path's byte for byte, and TCB_PLAIN_UPLOAD's single copy too."""
    torch = pytest.importorskip("torch")
    x = synth.small("sin_decay", (256, 128, 136), seed=11)  # 34 MiB: above the 32 MiB threshold
    prm = gpu_pkg.Params(target_re=1e-4)
    host = torch.from_numpy(x.reshape(-1).view(np.uint8)).pin_memory()
    src = gpu_pkg.SourceBuffer(memoryview(host.numpy()), gpu_pkg.Dtype.float64, list(x.shape))
    a = gpu_pkg.compress(src, prm).container
    dev = host.to("cuda")
    torch.cuda.synchronize()
    b = gpu_pkg.compress_device(dev.data_ptr(), x.nbytes, gpu_pkg.Dtype.float64, x.shape, prm).container
    assert a == b
    ref = oracle.compress(x, target_re=1e-4)
    assert gpu_pkg.compress(gpu_pkg.SourceBuffer.from_array(x), prm).container == a  # pageable: single copy
    assert abs(len(a) - len(ref.container)) <= 0.01 * len(ref.container)


@pytest.mark.parametrize("dtype,shape", [(np.float32, (300, 512, 640)), (np.float64, (256, 512, 520)),
                                          (np.float32, (1000, 256, 1024))])
def test_row_slab_upload_ozaki_gram_is_bitwise(gpu_pkg, dtype, shape):
    """Pinned uploads whose first unfolding takes the Ozaki Gram arrive in row
    slabs, each slab's digits and complete product tiles running while the
    next is in flight (ragged last slab, rows not a tile multiple, 8 slabs):
    the container equals the device-resident path's byte for byte."""
    torch = pytest.importorskip("torch")
    x = np.random.default_rng(3).standard_normal(shape).astype(dtype)
    x *= np.exp(-np.arange(shape[0]) / 40.0).astype(dtype)[:, None, None]
    prm = gpu_pkg.Params(target_re=1e-2)
    dt = gpu_pkg.Dtype.float32 if dtype == np.float32 else gpu_pkg.Dtype.float64
    host = torch.from_numpy(x.reshape(-1).view(np.uint8)).pin_memory()
    src = gpu_pkg.SourceBuffer(memoryview(host.numpy()), dt, list(x.shape))
    a = gpu_pkg.compress(src, prm)
    dev = host.to("cuda")
    torch.cuda.synchronize()
    b = gpu_pkg.compress_device(dev.data_ptr(), x.nbytes, dt, x.shape, prm)
    assert a.ranks == b.ranks
    assert a.container == b.container


def test_eig_large_cluster_cholqr(gpu_pkg):
    """A mode whose kept eigenvalues include a big noise-floor cluster (c3's
    500-row modes): the cluster is orthonormalised by CholQR2 (MGS only on a
    breakdown); the vectors stay orthonormal to roundoff, the strong directions
    match LAPACK's subspace, and every kept pair has a small residual."""
    rng = np.random.default_rng(5)
    n, k, r = 300, 1200, 280
    b = rng.standard_normal((n, k)) * np.where(np.arange(k) < 24, 1.0, 1e-4)
    g = b @ b.T
    ev, u = gpu_pkg.eig(g, r)
    lam, vec = np.linalg.eigh(g)
    lam, vec = lam[::-1], vec[:, ::-1]
    assert np.max(np.abs(ev - lam)) <= 1e-12 * lam[0] * np.sqrt(n)
    assert np.max(np.abs(u.T @ u - np.eye(r))) < 1e-12
    # strong directions: principal-angle sine against LAPACK
    s = np.linalg.svd(vec[:, :24].T @ u[:, :24], compute_uv=False)
    assert np.sqrt(max(0.0, 1 - s.min() ** 2)) < 1e-6
    res = np.linalg.norm(g @ u - u * ev[:r], axis=0)
    assert res.max() <= 1e-9 * lam[0]
