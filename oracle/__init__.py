"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes bindings over ``oracle/liboracle.so``: a plain C++ restatement of the
reference compress path (ATC ``tucomp``, /root/reference/proj).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline and
``--impl reference``) may import this package, and only as the checker or the
timed CPU baseline — never on the product path.

Pinning: the integer/bitstream half is checked bit-for-bit against the
reference's own sources compiled verbatim into ``oracle/_ref`` (see
``oracle/ref.py``); the floating-point half (Gram, eigensolver, SVD, TTM,
Householder) restates Eigen's algorithms and is pinned against numpy/LAPACK
("parity unpinned" with respect to Eigen itself, which is absent here).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

DTYPES = {
    np.dtype(np.int8): 0, np.dtype(np.uint8): 1, np.dtype(np.int16): 2, np.dtype(np.uint16): 3,
    np.dtype(np.int32): 4, np.dtype(np.uint32): 5, np.dtype(np.int64): 6, np.dtype(np.uint64): 7,
    np.dtype(np.float32): 8, np.dtype(np.float64): 9,
}


class OracleError(RuntimeError):
    pass


class Params(C.Structure):
    _fields_ = [
        ("has_re", C.c_int), ("re", C.c_double), ("has_sse", C.c_int), ("sse", C.c_double),
        ("rtmss", C.c_double), ("coder", C.c_int), ("split", C.c_int), ("simple", C.c_int),
        ("f32", C.c_int), ("backend", C.c_int), ("block", C.c_uint64),
        ("has_storage", C.c_int), ("storage", C.c_uint64 * 8),
        ("has_mode", C.c_int), ("mode", C.c_uint64 * 8), ("method", C.c_int),
    ]


class _Result(C.Structure):
    _fields_ = [
        ("container", C.POINTER(C.c_uint8)), ("size", C.c_uint64),
        ("norm_sq", C.c_double), ("target_sse", C.c_double), ("trunc", C.c_double),
        ("core_quant", C.c_double), ("estimate", C.c_double),
        ("factor_terms", C.c_double * 8), ("ranks", C.c_uint64 * 8), ("d", C.c_int),
        ("core_last_plane", C.c_int), ("core_k", C.c_int), ("precision_loss", C.c_int),
        ("original_bytes", C.c_uint64),
        ("t_sthosvd", C.c_double), ("t_quant", C.c_double), ("t_core", C.c_double),
        ("t_factor", C.c_double), ("t_ser", C.c_double), ("t_total", C.c_double),
    ]


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise OracleError(f"{path} missing: run __graft_entry__.build() (or make -C oracle)")
        L = C.CDLL(path)
        L.orc_last_error.restype = C.c_char_p
        for name in ("orc_sum_sq_f64", "orc_sum_sq_f32", "orc_backward_sq"):
            getattr(L, name).restype = C.c_double
        _LIB = L
    return _LIB


def _check(rc):
    if rc != 0:
        raise OracleError(lib().orc_last_error().decode())


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _take(ptr, n, ctype, dtype):
    if n == 0:
        out = np.zeros(0, dtype)
    else:
        out = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ctype)), shape=(n,)).astype(dtype, copy=True)
    lib().orc_free(C.cast(ptr, C.c_void_p))
    return out


def make_params(target_re=None, target_sse=None, rtmss=0.5, coder=0, split=True, simple=False,
                internal_float32=False, backend=0, block_size=0, storage_order=None, mode_order=None, method=0):
    p = Params()
    p.method = int(method)
    p.has_re = int(target_re is not None)
    p.re = float(target_re or 0.0)
    p.has_sse = int(target_sse is not None)
    p.sse = float(target_sse or 0.0)
    p.rtmss = rtmss
    p.coder = coder
    p.split = int(split)
    p.simple = int(simple)
    p.f32 = int(internal_float32)
    p.backend = backend
    p.block = block_size
    if storage_order is not None:
        p.has_storage = 1
        for i, v in enumerate(storage_order):
            p.storage[i] = v
    if mode_order is not None:
        p.has_mode = 1
        for i, v in enumerate(mode_order):
            p.mode[i] = v
    return p


@dataclass
class CompressInfo:
    container: bytes
    norm_sq: float
    target_sse: float
    truncation_sse: float
    core_quant_sse: float
    estimate_sse: float
    factor_terms: list
    ranks: list
    core_last_plane: int
    core_k: int
    precision_loss: bool
    original_bytes: int
    times_ms: dict = field(default_factory=dict)


def compress(data: np.ndarray, skip_bytes: bytes = b"", **kw) -> CompressInfo:
    """Restated ``tucomp::pipeline::compress`` (pipeline.cpp:240-252)."""
    data = np.ascontiguousarray(data)
    raw = skip_bytes + data.tobytes()
    buf = np.frombuffer(raw, dtype=np.uint8) if raw else np.zeros(1, np.uint8)
    shape = np.asarray(data.shape, dtype=np.uint64)
    res = _Result()
    _check(lib().orc_compress(_p(buf), C.c_uint64(len(raw)), DTYPES[data.dtype], _p(shape), len(data.shape),
                              C.c_uint64(len(skip_bytes)), C.byref(make_params(**kw)), C.byref(res)))
    d = res.d
    cont = bytes(_take(res.container, res.size, C.c_uint8, np.uint8))
    return CompressInfo(
        container=cont, norm_sq=res.norm_sq, target_sse=res.target_sse, truncation_sse=res.trunc,
        core_quant_sse=res.core_quant, estimate_sse=res.estimate,
        factor_terms=[res.factor_terms[i] for i in range(d)], ranks=[int(res.ranks[i]) for i in range(d)],
        core_last_plane=res.core_last_plane, core_k=res.core_k, precision_loss=bool(res.precision_loss),
        original_bytes=res.original_bytes,
        times_ms=dict(sthosvd=res.t_sthosvd, quantize=res.t_quant, core_encode=res.t_core,
                      factor_encode=res.t_factor, serialize=res.t_ser, total=res.t_total))


def decompress(container: bytes, shape, internal_float32=False) -> np.ndarray:
    buf = np.frombuffer(container, dtype=np.uint8)
    ptr = C.c_void_p()
    n = C.c_uint64()
    fn = lib().orc_decompress_f32 if internal_float32 else lib().orc_decompress_f64
    _check(fn(_p(buf), C.c_uint64(len(container)), C.byref(ptr), C.byref(n)))
    ct = C.c_float if internal_float32 else C.c_double
    dt = np.float32 if internal_float32 else np.float64
    return _take(ptr, n.value, ct, dt).reshape(shape)


def sthosvd(x: np.ndarray, target: float, order=None, backend=0) -> dict:
    x = np.ascontiguousarray(x, dtype=np.float64)
    d = x.ndim
    shape = np.asarray(x.shape, np.uint64)
    core = C.c_void_p()
    core_shape = (C.c_uint64 * d)()
    facs = (C.c_void_p * d)()
    ranks = (C.c_uint64 * d)()
    trunc = (C.c_double * d)()
    s2 = (C.c_void_p * d)()
    s2n = (C.c_uint64 * d)()
    ordo = (C.c_uint64 * d)()
    oarr = None
    if order is not None:
        oarr = np.asarray(order, np.uint64)
    _check(lib().orc_sthosvd_f64(_p(x), _p(shape), d, C.c_double(target),
                                 _p(oarr) if oarr is not None else None, backend, C.byref(core), core_shape,
                                 facs, ranks, trunc, s2, s2n, ordo))
    cs = [int(core_shape[i]) for i in range(d)]
    out = dict(core=_take(core, int(np.prod(cs)), C.c_double, np.float64).reshape(cs),
               ranks=[int(ranks[i]) for i in range(d)], trunc=[trunc[i] for i in range(d)],
               order=[int(ordo[i]) for i in range(d)])
    out["factors"] = [_take(facs[i], x.shape[i] * out["ranks"][i], C.c_double, np.float64)
                      .reshape(x.shape[i], out["ranks"][i]) for i in range(d)]
    out["sigma2"] = [_take(s2[i], int(s2n[i]), C.c_double, np.float64) for i in range(d)]
    return out


def eig(a: np.ndarray):
    """SelfAdjointEigenSolver stand-in: ascending eigenvalues, eigenvector columns."""
    n = a.shape[0]
    m = np.asfortranarray(a, dtype=np.float64).copy(order="F")
    ev = np.zeros(n)
    flat = m.reshape(-1, order="F").copy()
    _check(lib().orc_eig_f64(_p(flat), C.c_uint64(n), _p(ev)))
    return ev, flat.reshape((n, n), order="F")


def quantize(core: np.ndarray, method: int = 0):
    """corecodec::quantize (core_codec.cpp:55-93) under vectorize::Method `method`."""
    core = np.ascontiguousarray(core, dtype=np.float64)
    n = core.size
    shape = np.asarray(core.shape, np.uint64)
    mag = np.zeros(n, np.uint64)
    neg = np.zeros(n, np.uint8)
    k = C.c_int()
    zero = C.c_int()
    sn = np.zeros(int(sum(core.shape)), np.float64)
    _check(lib().orc_quantize_method_f64(_p(core), _p(shape), core.ndim, int(method), _p(mag), _p(neg), C.byref(k),
                                         C.byref(zero), _p(sn)))
    parts, o = [], 0
    for e in core.shape:
        parts.append(sn[o:o + e].copy())
        o += e
    return mag, neg, k.value, bool(zero.value), parts


def encode(mag, neg, target_int, coder=0, block_size=0, split=True, fixed_plane=-1):
    """Encoder::plan + finalize; returns (stream section bytes, last_plane, achieved_sse_int, decoded)."""
    mag = np.ascontiguousarray(mag, np.uint64)
    neg = np.ascontiguousarray(neg, np.uint8)
    n = mag.size
    out = C.c_void_p()
    ln = C.c_uint64()
    lp = C.c_int()
    ach = C.c_double()
    dec = np.zeros(max(n, 1), np.uint64)
    _check(lib().orc_encode(_p(mag), _p(neg), C.c_uint64(n), C.c_double(target_int), coder,
                            C.c_uint64(block_size), int(split), fixed_plane, C.byref(out), C.byref(ln),
                            C.byref(lp), C.byref(ach), _p(dec)))
    return bytes(_take(out, ln.value, C.c_uint8, np.uint8)), lp.value, ach.value, dec[:n]


def encode_symbols(coder, syms) -> bytes:
    s = np.ascontiguousarray(syms, np.uint64)
    out = C.c_void_p()
    ln = C.c_uint64()
    _check(lib().orc_encode_symbols(coder, _p(s) if s.size else None, C.c_uint64(s.size), C.byref(out),
                                    C.byref(ln)))
    return bytes(_take(out, ln.value, C.c_uint8, np.uint8))


def decode_symbols(payload: bytes) -> np.ndarray:
    b = np.frombuffer(payload, np.uint8)
    out = C.c_void_p()
    n = C.c_uint64()
    _check(lib().orc_decode_symbols(_p(b), C.c_uint64(len(payload)), C.byref(out), C.byref(n)))
    return _take(out, n.value, C.c_uint64, np.uint64)


def encode_factor(u, dead, slice_norms, coder=0, simple=False, core_step_log2=0, term_cap=0.0):
    u = np.ascontiguousarray(u, np.float64)
    n, r = u.shape
    dead = np.ascontiguousarray(dead, np.uint8)
    sn = np.ascontiguousarray(slice_norms, np.float64)
    out = C.c_void_p()
    ln = C.c_uint64()
    k = C.c_int()
    cnt = C.c_uint64()
    flips = np.zeros(max(r, 1), np.int8)
    term = C.c_double()
    plane = C.c_int()
    dec = np.zeros(n * r, np.float64)
    _check(lib().orc_encode_factor_f64(_p(u), C.c_uint64(n), C.c_uint64(r), _p(dead), _p(sn), coder, int(simple),
                                       core_step_log2, C.c_double(term_cap), C.byref(out), C.byref(ln),
                                       C.byref(k), C.byref(cnt), _p(flips), C.byref(term), C.byref(plane),
                                       _p(dec)))
    return dict(stream=bytes(_take(out, ln.value, C.c_uint8, np.uint8)), k=k.value, count=cnt.value,
                flips=flips[:r], term=term.value, plane=plane.value, decoded=dec.reshape(n, r))


def sum_sq(x: np.ndarray) -> float:
    x = np.ascontiguousarray(x)
    if x.dtype == np.float32:
        return lib().orc_sum_sq_f32(_p(x), C.c_uint64(x.size))
    x = x.astype(np.float64, copy=False)
    return lib().orc_sum_sq_f64(_p(x), C.c_uint64(x.size))


def backward_sq(m) -> float:
    m = np.ascontiguousarray(m, np.uint64)
    return lib().orc_backward_sq(_p(m), C.c_uint64(m.size))


def pick_rank(s2, budget):
    s2 = np.ascontiguousarray(s2, np.float64)
    r = C.c_uint64()
    dis = C.c_double()
    _check(lib().orc_pick_rank(_p(s2), C.c_uint64(s2.size), C.c_double(budget), C.byref(r), C.byref(dis)))
    return r.value, dis.value


def alpha_weights(sn, n):
    sn = np.ascontiguousarray(sn, np.float64)
    out = np.zeros(sn.size)
    _check(lib().orc_alpha_weights(_p(sn), C.c_uint64(sn.size), C.c_uint64(n), _p(out)))
    return out


def transpose(x: np.ndarray, perm):
    x = np.ascontiguousarray(x, np.float64)
    shape = np.asarray(x.shape, np.uint64)
    p = np.asarray(perm, np.uint64)
    out = np.zeros(x.size)
    _check(lib().orc_transpose_f64(_p(x), _p(shape), x.ndim, _p(p), _p(out)))
    return out.reshape([x.shape[i] for i in perm])


def threads() -> int:
    """Host threads the oracle's OpenMP loops use (results do not depend on it)."""
    return int(lib().orc_threads())


def order_map(method: int, shape) -> np.ndarray:
    """vectorize::OrderMap::build (vectorize.cpp:163-170): flat position of each coefficient."""
    sh = np.asarray(shape, np.uint64)
    out = np.empty(int(np.prod(sh)), np.uint64)
    _check(lib().orc_order_map(int(method), _p(sh), len(sh), _p(out)))
    return out
