"""Device decompress (pipeline::decompress / decompress_tensor) against the
oracle's decoder on the same containers: the stream decode is integer work and
must reproduce the oracle exactly (checked through the reconstruction at fp64
roundoff), the TTM expansions are floating point (tolerance), the dtype emit
follows cast_out (container.cpp:98-140)."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("kind,shape,re", [("sin_decay", (48, 40, 36), 1e-4), ("sin", (32, 32, 32), 1e-3),
                                           ("blobs", (40, 30, 20), 1e-2), ("random", (20, 16, 12), 1e-1),
                                           ("sin_decay", (96, 64, 80), 1e-6)])
def test_decompress_gpu_containers(gpu_pkg, kind, shape, re):
    x = synth.small(kind, shape, seed=2)
    res = gpu_pkg.compress(gpu_pkg.SourceBuffer.from_array(x), gpu_pkg.Params(target_re=re))
    ref = oracle.decompress(res.container, shape)
    got = gpu_pkg.decompress_tensor(res.container)
    assert got.shape == tuple(shape)
    assert _rel(got, ref) < 1e-12
    out = gpu_pkg.decompress(res.container)
    assert out.dtype == gpu_pkg.Dtype.float64 and out.shape == tuple(shape)
    assert _rel(out.to_array(), ref) < 1e-12


@pytest.mark.parametrize("opts", [dict(coder=1), dict(split=False), dict(simple=True), dict(block_size=256),
                                  dict(coder=1, split=False, block_size=512), dict(storage_order=(2, 0, 1)),
                                  dict(method=1), dict(method=2, block_size=512)])
def test_decompress_oracle_containers(gpu_pkg, opts):
    """Containers written by the oracle (rANS, non-split, simple weights, multi-block
    streams, a non-default storage order): every decode path on the device."""
    shape = (40, 36, 28)
    x = synth.small("sin_decay", shape, seed=4)
    info = oracle.compress(x, target_re=1e-4, **opts)
    ref = oracle.decompress(info.container, shape)
    got = gpu_pkg.decompress_tensor(info.container)
    assert _rel(got, ref) < 1e-12


@pytest.mark.parametrize("dtype", [np.uint16, np.int16, np.uint8, np.int32, np.float32])
def test_decompress_emit_dtypes(gpu_pkg, dtype):
    shape = (32, 24, 20)
    base = synth.small("blobs", shape, seed=6)
    if np.issubdtype(dtype, np.integer):
        info = np.iinfo(dtype)
        lo, hi = max(info.min, -3000), min(info.max, 3000)
        x = np.clip(np.round((base - base.min()) / np.ptp(base) * (hi - lo) + lo), info.min, info.max).astype(dtype)
    else:
        x = base.astype(dtype)
    res = gpu_pkg.compress(gpu_pkg.SourceBuffer.from_array(x), gpu_pkg.Params(target_re=1e-3))
    out = gpu_pkg.decompress(res.container)
    assert out.dtype == gpu_pkg.Dtype(oracle.DTYPES[np.dtype(dtype)]) and out.shape == shape
    y = out.to_array()
    ref = oracle.decompress(res.container, shape)
    if np.issubdtype(dtype, np.integer):
        info = np.iinfo(dtype)
        want = np.clip(np.rint(ref), info.min, info.max).astype(dtype)
        diff = np.abs(y.astype(np.int64) - want.astype(np.int64))
        assert diff.max() <= 1  # a rounding tie may flip under fp64 roundoff
        assert np.mean(diff == 0) > 0.999
    else:
        assert np.allclose(y, ref.astype(dtype), rtol=1e-6, atol=1e-6 * np.max(np.abs(ref)))


def test_decompress_zero_tensor(gpu_pkg):
    x = np.zeros((8, 6, 4))
    res = gpu_pkg.compress(gpu_pkg.SourceBuffer.from_array(x), gpu_pkg.Params(target_re=1e-3))
    assert np.all(gpu_pkg.decompress_tensor(res.container) == 0)


def test_decompress_errors(gpu_pkg):
    x = synth.small("sin", (16, 16, 16), seed=1)
    c = gpu_pkg.compress(gpu_pkg.SourceBuffer.from_array(x), gpu_pkg.Params(target_re=1e-3)).container
    with pytest.raises(gpu_pkg.TucompError, match="container: bad magic"):
        gpu_pkg.decompress(b"XXXX" + c[4:])
    with pytest.raises(gpu_pkg.TucompError, match="container: truncated"):
        gpu_pkg.decompress(c[: len(c) // 2])


def _patch(c, off, val):
    b = bytearray(c)
    b[off:off + len(val)] = val
    return bytes(b)


@pytest.mark.parametrize("off,val,msg", [
    (4, b"\x02", "container: unsupported format version 2"),
    (5, b"\x0c", "container: unknown source dtype"),
    (8, b"\x02", "container: unknown entropy coder id"),
    (9, b"\x03", "container: unknown vectorization method id"),
    (60, b"\x00\x00", "container: corrupt mode permutations"),   # processing order (0,0,..)
    (63, b"\x03", "container: corrupt mode permutations"),       # storage order entry out of range
    (36, (0).to_bytes(8, "little"), "container: corrupt mode sizes or ranks"),   # rank 0
    (36, (17).to_bytes(8, "little"), "container: corrupt mode sizes or ranks"),  # rank > size
    (12, (0).to_bytes(8, "little"), "container: corrupt mode sizes or ranks"),   # size 0
])
def test_decompress_header_validation(gpu_pkg, off, val, msg):
    """Header checks of read_container (reference container.cpp:338-420), byte
    offsets per the layout in container.cpp write_container: magic[0:4] version[4]
    dtype[5] f32[6] d[7] coder[8] method[9] flags[10] pad[11] sizes[12:36]
    ranks[36:60] processing order[60:63] storage order[63:66] for d=3."""
    x = synth.small("sin", (16, 16, 16), seed=1)
    c = gpu_pkg.compress(gpu_pkg.SourceBuffer.from_array(x), gpu_pkg.Params(target_re=1e-3)).container
    assert c[7] == 3
    with pytest.raises(gpu_pkg.TucompError, match=msg):
        gpu_pkg.decompress(_patch(c, off, val))


@pytest.mark.parametrize("dtype", [np.float64, np.uint16])
def test_decompress_into_device_memory(gpu_pkg, dtype):
    """tcb_decompress_device writes the same source-dtype bytes as
    tcb_decompress, into a caller device buffer; a short buffer is an error."""
    torch = pytest.importorskip("torch")
    shape = (40, 32, 24)
    base = synth.small("blobs", shape, seed=9)
    x = (np.round((base - base.min()) / np.ptp(base) * 4000).astype(dtype) if dtype != np.float64 else base)
    c = gpu_pkg.compress(gpu_pkg.SourceBuffer.from_array(x), gpu_pkg.Params(target_re=1e-3)).container
    host = gpu_pkg.decompress(c)
    out = torch.empty(x.nbytes, dtype=torch.uint8, device="cuda")
    dt, sh, _ = gpu_pkg.decompress_device(c, out.data_ptr(), x.nbytes)
    assert dt == host.dtype and sh == shape
    assert out.cpu().numpy().tobytes() == host.bytes
    with pytest.raises(gpu_pkg.TucompError, match="output buffer holds"):
        gpu_pkg.decompress_device(c, out.data_ptr(), x.nbytes - 1)
