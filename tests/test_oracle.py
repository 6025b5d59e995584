"""CPU tests of the oracle (test infrastructure): pinned against the golden
vectors produced by the reference's own sources (tests/golden/golden.json),
against the live verbatim-reference build when present (oracle/_ref), against
SPEC.md's known-answer examples, and against numpy/LAPACK for the FP half."""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle
import oracle.ref as R
import synth

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
need_ref = pytest.mark.skipif(not R.available(), reason="oracle/_ref (verbatim reference build) not present")


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def core_like(shape, seed, decay):
    rng = np.random.default_rng(seed)
    idx = np.indices(shape).sum(0).astype(np.float64)
    return rng.standard_normal(shape) * np.exp(-decay * idx / idx.max())


# ---------------------------------------------------------------- golden pins
@pytest.mark.parametrize("g", GOLDEN["symbols"], ids=lambda g: f"case{g['case']}-coder{g['coder']}")
def test_entropy_matches_golden(g):
    assert oracle.encode_symbols(g["coder"], g["symbols"]).hex() == g["bytes"]
    if g["symbols"]:
        assert oracle.decode_symbols(bytes.fromhex(g["bytes"])).tolist() == g["symbols"]


@pytest.mark.parametrize("g", GOLDEN["quantize"], ids=lambda g: f"seed{g['seed']}")
def test_quantize_matches_golden(g):
    mag, neg, k, zero, sn = oracle.quantize(core_like(tuple(g["shape"]), g["seed"], g["decay"]))
    assert k == g["k"] and zero == g["zero"]
    assert sha(mag.tobytes()) == g["mag_sha"] and sha(neg.tobytes()) == g["neg_sha"]
    assert [[float(v).hex() for v in ax] for ax in sn] == g["slice_norms_hex"]


@pytest.mark.parametrize("g", GOLDEN["encode"],
                         ids=lambda g: f"s{g['seed']}-f{g['frac']}-c{g['coder']}-sp{int(g['split'])}-fx{g['fixed']}")
def test_encoder_matches_golden(g):
    mag, neg, k, _, _ = oracle.quantize(core_like(tuple(g["shape"]), g["seed"], g["decay"]))
    tot = float((mag.astype(np.float64) ** 2).sum())
    s, lp, ach, dec = oracle.encode(mag, neg, tot * g["frac"], coder=g["coder"], split=g["split"],
                                    fixed_plane=g["fixed"])
    assert lp == g["last_plane"] and len(s) == g["len"] and sha(s) == g["sha"]
    assert float(ach).hex() == g["achieved_hex"] and sha(dec.tobytes()) == g["dec_sha"]


@pytest.mark.parametrize("g", GOLDEN["sum_squares"], ids=lambda g: f"{g['dtype']}-{g['n']}")
def test_sum_squares_matches_golden_bitwise(g):
    x = np.random.default_rng(g["n"]).uniform(-3, 3, g["n"])
    if g["dtype"] == "float32":
        x = x.astype(np.float32)
    assert float(oracle.sum_sq(x)).hex() == g["value_hex"]


# ---------------------------------------------------------------- live verbatim reference
@need_ref
@pytest.mark.parametrize("seed", range(3))
def test_encoder_matches_live_reference(seed):
    core = core_like((18, 30, 25), 100 + seed, 6.0)
    mag, neg, k, zero, sn = oracle.quantize(core)
    m2, n2, k2, z2, sn2 = R.quantize(core)
    assert np.array_equal(mag, m2) and np.array_equal(neg, n2) and k == k2
    tot = float((mag.astype(np.float64) ** 2).sum())
    for frac in (3e-2, 1e-5, 1e-10):
        for workers in (1, 4):
            a = oracle.encode(mag, neg, tot * frac)
            b = R.encode(mag, neg, tot * frac, workers=workers)
            assert a[0] == b[0] and a[1] == b[1] and a[2] == b[2]


@need_ref
def test_container_bytes_roundtrip_through_reference_reader_writer():
    x = synth.small("sin", (24, 20, 16), seed=4)
    info = oracle.compress(x, target_re=1e-3)
    assert R.container_rewrite(info.container) == info.container
    mag, neg = R.container_core(info.container)
    assert mag.size == int(np.prod(info.ranks))


# ---------------------------------------------------------------- SPEC.md known answers
def test_rank_rule_examples():
    assert oracle.pick_rank([100, 9, 4, 1], 5) == (2, 5.0)
    assert oracle.pick_rank([100, 0, 0], 1)[0] == 1
    assert oracle.pick_rank([3, 2, 1], 0) == (3, 0.0)


def test_quantize_example():
    mag, neg, k, zero, _ = oracle.quantize(np.array([[[0.5, -0.25]]]))
    assert k == 64 and mag.tolist() == [2 ** 63, 2 ** 62] and neg.tolist() == [0, 1]


def test_alpha_weight_example():
    assert oracle.alpha_weights([2.0], 1)[0] == pytest.approx(3 * 4.0)  # SPEC.md:436-438 (n=r=1 -> 3 sigma^2)


def test_rle_example():
    # column 00101 -> runs (2, 1, 0); observed through the coder round trip
    runs = [2, 1, 0]
    assert oracle.decode_symbols(oracle.encode_symbols(0, runs)).tolist() == runs


def test_mode_orders():
    x = np.zeros((5, 3, 4)) + 1.0
    f = oracle.sthosvd(x, 0.0)
    assert f["order"] == [1, 2, 0]  # stable ascending by extent (sthosvd.cpp:28-33)


# ---------------------------------------------------------------- FP half vs numpy/LAPACK
@pytest.mark.parametrize("n", [1, 2, 5, 40, 128])
def test_eigensolver_vs_lapack(n):
    b = np.random.default_rng(n).standard_normal((n, 2 * n + 3))
    g = b @ b.T
    ev, vec = oracle.eig(g)
    w = np.linalg.eigvalsh(g)
    assert np.allclose(ev, w, rtol=0, atol=1e-12 * abs(w).max())
    assert np.abs(vec.T @ vec - np.eye(n)).max() < 1e-12
    assert np.abs(g @ vec - vec * ev).max() < 1e-10 * abs(w).max()


def test_sthosvd_zero_target_is_lossless():
    x = synth.small("random", (6, 7, 8), seed=2)
    f = oracle.sthosvd(x, 0.0)
    assert f["ranks"] == [6, 7, 8]
    core = f["core"]
    # reconstruct: X = core x_i U_i in processing order
    y = np.einsum("abc,ia,jb,kc->ijk", core, *[f["factors"][m] for m in f["order"]])
    y = np.transpose(y, np.argsort(f["order"]))
    assert np.abs(y - x).max() < 1e-10


def test_sthosvd_rank_one():
    u, v, w = (np.random.default_rng(s).standard_normal(n) for s, n in ((1, 9), (2, 10), (3, 11)))
    x = np.einsum("i,j,k->ijk", u, v, w)
    f = oracle.sthosvd(x, 1e-6 * float((x ** 2).sum()))
    assert f["ranks"] == [1, 1, 1] and sum(f["trunc"]) < 1e-12 * float((x ** 2).sum())


def test_sthosvd_truncation_equals_discarded_energy():
    x = synth.small("sin_decay", (16, 18, 20), seed=3)
    tgt = 1e-4 * float((x ** 2).sum())
    f = oracle.sthosvd(x, tgt)
    core = f["core"]
    y = np.einsum("abc,ia,jb,kc->ijk", core, *[f["factors"][m] for m in f["order"]])
    y = np.transpose(y, np.argsort(f["order"]))
    assert float(((y - x) ** 2).sum()) == pytest.approx(sum(f["trunc"]), rel=1e-6)
    assert sum(f["trunc"]) <= tgt


def test_transpose_roundtrip():
    x = synth.small("random", (3, 4, 5), seed=1)
    p = [2, 0, 1]
    t = oracle.transpose(x, p)
    assert np.array_equal(t, np.transpose(x, p))


# ---------------------------------------------------------------- pipeline behaviour
@pytest.mark.parametrize("kind,shape,re", [("sin", (32, 32, 32), 1e-3), ("blobs", (20, 30, 25), 1e-2),
                                          ("sin_decay", (24, 24, 24), 1e-5)])
def test_compress_roundtrip_meets_target(kind, shape, re):
    x = synth.small(kind, shape, seed=5)
    info = oracle.compress(x, target_re=re)
    y = oracle.decompress(info.container, shape)
    err = np.sqrt(((y - x) ** 2).sum() / (x ** 2).sum())
    assert err <= re * 1.05
    assert info.estimate_sse == pytest.approx(((y - x) ** 2).sum(), rel=0.2)


def test_internal_float32_throws_like_reference():
    """The reference's factorize() checks U^T U - I in float against 1e-8
    (factor_codec.cpp:29-31), so any factor with >= 2 columns throws."""
    x = synth.small("sin", (32, 32, 32), seed=1, dtype=np.float32)
    with pytest.raises(oracle.OracleError, match="not orthonormal"):
        oracle.compress(x, target_re=1e-3, internal_float32=True)


def test_error_messages():
    x = np.ones((4, 4, 4))
    with pytest.raises(oracle.OracleError, match="mutually exclusive"):
        oracle.compress(x, target_re=1e-2, target_sse=1.0)
    with pytest.raises(oracle.OracleError, match="no error target"):
        oracle.compress(x)
    x[0, 0, 0] = np.inf
    with pytest.raises(oracle.OracleError, match="non-finite"):
        oracle.compress(x, target_re=1e-2)


def test_zero_tensor_container():
    info = oracle.compress(np.zeros((4, 5, 6)), target_re=1e-2)
    assert info.container[:4] == b"TKC1"
    y = oracle.decompress(info.container, (4, 5, 6))
    assert not y.any()


def test_uint16_source_precision_flag():
    x = (np.arange(4 * 5 * 6).reshape(4, 5, 6) % 17).astype(np.uint16)
    info = oracle.compress(x, target_re=1e-2)
    assert info.original_bytes == x.nbytes and not info.precision_loss
    big = np.full((4, 4, 4), 2 ** 60, np.int64)
    big[0, 0, 0] = 1
    assert oracle.compress(big, target_re=1e-2).precision_loss


# ---------------------------------------------------------------- vectorization methods
@pytest.mark.parametrize("shape", [(3, 4, 5), (13, 11, 7), (9, 6, 4, 3), (1, 8, 1), (17,)])
@pytest.mark.parametrize("method", [1, 2])
def test_order_map_matches_reference(shape, method):
    import oracle.ref as R

    if not R.available():
        pytest.skip("oracle/_ref not built")
    assert np.array_equal(oracle.order_map(method, shape), R.order_map(method, shape))


@pytest.mark.parametrize("method", [1, 2])
def test_quantize_method_matches_reference(method):
    import oracle.ref as R

    if not R.available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(method)
    core = rng.standard_normal((11, 9, 7)) * np.exp(-np.indices((11, 9, 7)).sum(0) / 4.0)
    mag, neg, k, zero, sn = oracle.quantize(core, method)
    rm, rn, rk, rz, rsn = R.quantize_method(core, method)
    assert k == rk and zero == rz and np.array_equal(mag, rm) and np.array_equal(neg, rn)
    assert np.concatenate(sn).tobytes() == rsn.tobytes()  # slice norms summed in vectorised order


@pytest.mark.parametrize("method", [1, 2])
def test_compress_method_round_trip(method):
    x = synth.small("sin_decay", (24, 20, 16), seed=3)
    info = oracle.compress(x, target_re=1e-3, method=method)
    assert info.container[9] == method  # header byte 9: vectorize::Method
    y = oracle.decompress(info.container, x.shape)
    assert np.linalg.norm(y - x) / np.linalg.norm(x) <= 1.05e-3


@pytest.mark.parametrize("off,val,msg", [
    (4, b"\x02", "container: unsupported format version 2"),
    (5, b"\x0c", "container: unknown source dtype"),
    (8, b"\x02", "container: unknown entropy coder id"),
    (9, b"\x03", "container: unknown vectorization method id"),
    (60, b"\x00\x00", "container: corrupt mode permutations"),
    (63, b"\x03", "container: corrupt mode permutations"),
    (36, (0).to_bytes(8, "little"), "container: corrupt mode sizes or ranks"),
    (36, (17).to_bytes(8, "little"), "container: corrupt mode sizes or ranks"),
])
def test_oracle_header_validation(off, val, msg):
    """The oracle's decoder rejects the headers read_container rejects
    (reference container.cpp:338-420), with the same messages."""
    x = synth.small("sin", (16, 16, 16), seed=1)
    c = bytearray(oracle.compress(x, target_re=1e-3).container)
    c[off:off + len(val)] = val
    with pytest.raises(oracle.OracleError, match=msg):
        oracle.decompress(bytes(c), (16, 16, 16))
    if R.available():  # pin: the reference's read_container gives the same message
        with pytest.raises(R.RefError, match=msg):
            R.container_rewrite(bytes(c))
