"""TEST INFRASTRUCTURE ONLY — probes over the reference's own integer sources.

``oracle/_ref/libtucomp_ref.so`` is compiled verbatim from
/root/reference/proj/src by ``oracle/ref/build_ref.sh`` (gitignored, travels to
the GPU box with the snapshot).  Tests skip when it is absent.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
PATH = os.path.join(_HERE, "_ref", "libtucomp_ref.so")
_LIB = None


class RefError(RuntimeError):
    pass


def available() -> bool:
    return os.path.exists(PATH)


def lib():
    global _LIB
    if _LIB is None:
        L = C.CDLL(PATH)
        L.ref_last_error.restype = C.c_char_p
        L.ref_backend.restype = C.c_char_p
        for n in ("ref_sum_squares_f64", "ref_sum_squares_f32", "ref_backward_sum"):
            getattr(L, n).restype = C.c_double
        _LIB = L
    return _LIB


def _check(rc):
    if rc != 0:
        raise RefError(lib().ref_last_error().decode())


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _take(ptr, n, ctype, dtype):
    out = (np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ctype)), shape=(n,)).astype(dtype, copy=True)
           if n else np.zeros(0, dtype))
    lib().ref_free(C.cast(ptr, C.c_void_p))
    return out


def encode(mag, neg, target_int, coder=0, block_size=0, split=True, fixed_plane=-1, workers=1):
    mag = np.ascontiguousarray(mag, np.uint64)
    neg = np.ascontiguousarray(neg, np.uint8)
    n = mag.size
    out = C.c_void_p()
    ln = C.c_uint64()
    lp = C.c_int()
    ach = C.c_double()
    dec = np.zeros(max(n, 1), np.uint64)
    _check(lib().ref_encode(_p(mag), _p(neg), C.c_uint64(n), C.c_double(target_int), coder, C.c_uint64(block_size),
                            int(split), fixed_plane, workers, C.byref(out), C.byref(ln), C.byref(lp),
                            C.byref(ach), _p(dec)))
    return bytes(_take(out, ln.value, C.c_uint8, np.uint8)), lp.value, ach.value, dec[:n]


def quantize(core: np.ndarray):
    core = np.ascontiguousarray(core, np.float64)
    n = core.size
    shape = np.asarray(core.shape, np.uint64)
    mag = np.zeros(n, np.uint64)
    neg = np.zeros(n, np.uint8)
    k = C.c_int()
    zero = C.c_int()
    sn = np.zeros(int(sum(core.shape)))
    _check(lib().ref_quantize_f64(_p(core), _p(shape), core.ndim, _p(mag), _p(neg), C.byref(k), C.byref(zero),
                                  _p(sn)))
    parts, o = [], 0
    for e in core.shape:
        parts.append(sn[o:o + e].copy())
        o += e
    return mag, neg, k.value, bool(zero.value), parts


def encode_symbols(coder, syms) -> bytes:
    s = np.ascontiguousarray(syms, np.uint64)
    out = C.c_void_p()
    ln = C.c_uint64()
    _check(lib().ref_encode_symbols(coder, _p(s) if s.size else None, C.c_uint64(s.size), C.byref(out),
                                    C.byref(ln)))
    return bytes(_take(out, ln.value, C.c_uint8, np.uint8))


def decode_symbols(payload: bytes):
    b = np.frombuffer(payload, np.uint8)
    out = C.c_void_p()
    n = C.c_uint64()
    _check(lib().ref_decode_symbols(_p(b), C.c_uint64(len(payload)), C.byref(out), C.byref(n)))
    return _take(out, n.value, C.c_uint64, np.uint64)


def container_rewrite(cont: bytes) -> bytes:
    b = np.frombuffer(cont, np.uint8)
    out = C.c_void_p()
    ln = C.c_uint64()
    _check(lib().ref_container_rewrite(_p(b), C.c_uint64(len(cont)), C.byref(out), C.byref(ln)))
    return bytes(_take(out, ln.value, C.c_uint8, np.uint8))


def container_core(cont: bytes):
    b = np.frombuffer(cont, np.uint8)
    mag = C.c_void_p()
    neg = C.c_void_p()
    n = C.c_uint64()
    _check(lib().ref_container_core(_p(b), C.c_uint64(len(cont)), C.byref(mag), C.byref(neg), C.byref(n)))
    return _take(mag, n.value, C.c_uint64, np.uint64), _take(neg, n.value, C.c_uint8, np.uint8)


def sum_sq(x: np.ndarray) -> float:
    x = np.ascontiguousarray(x)
    if x.dtype == np.float32:
        return lib().ref_sum_squares_f32(_p(x), C.c_uint64(x.size))
    return lib().ref_sum_squares_f64(_p(x.astype(np.float64, copy=False)), C.c_uint64(x.size))


def backward_sum(m) -> float:
    m = np.ascontiguousarray(m, np.uint64)
    return lib().ref_backward_sum(_p(m), C.c_uint64(m.size))


def backend() -> str:
    return lib().ref_backend().decode()


def order_map(method: int, shape) -> np.ndarray:
    """The reference's own vectorize::OrderMap::build (vectorize.cpp:163-170)."""
    sh = np.asarray(shape, np.uint64)
    out = np.empty(int(np.prod(sh)), np.uint64)
    _check(lib().ref_order_map(int(method), sh.ctypes.data_as(C.c_void_p), len(sh), out.ctypes.data_as(C.c_void_p)))
    return out


def quantize_method(core: np.ndarray, method: int):
    """The reference's corecodec::quantize under a vectorization method: (mag, neg, k, zero, slice norms)."""
    core = np.ascontiguousarray(core, np.float64)
    sh = np.asarray(core.shape, np.uint64)
    n = core.size
    mag = np.zeros(n, np.uint64)
    neg = np.zeros(n, np.uint8)
    k, zero = C.c_int(), C.c_int()
    sn = np.zeros(int(sh.sum()), np.float64)
    _check(lib().ref_quantize_method_f64(core.ctypes.data_as(C.c_void_p), sh.ctypes.data_as(C.c_void_p), core.ndim,
                                         int(method), mag.ctypes.data_as(C.c_void_p), neg.ctypes.data_as(C.c_void_p),
                                         C.byref(k), C.byref(zero), sn.ctypes.data_as(C.c_void_p)))
    return mag, neg, k.value, bool(zero.value), sn
