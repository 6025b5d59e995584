"""B200-native ATC compress path behind the reference's pipeline API.

Python mirror of ``tucomp::pipeline`` (/root/reference/proj/include/tucomp/
pipeline.hpp:14-71) over the C ABI in ``include/tucomp_b200.h``
(``libtucomp_b200.so``, hand-written sm_100a CUDA).  Names, argument meaning
and error text follow the reference: ``compress(SourceBuffer, Params)``
returns a ``CompressResult`` whose ``container`` bytes are the reference's
TKC1 format.  There is no CPU fallback: importing works anywhere (so the
library can be inspected), every compute call runs CUDA kernels and raises
``TucompError`` when the extension or a GPU is missing.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtucomp_b200.so")
_LIB = None


class TucompError(RuntimeError):
    """tucomp::Error (tensor.hpp:14-17)."""


class Dtype(enum.IntEnum):  # container::Dtype (container.hpp:16-27)
    int8 = 0
    uint8 = 1
    int16 = 2
    uint16 = 3
    int32 = 4
    uint32 = 5
    int64 = 6
    uint64 = 7
    float32 = 8
    float64 = 9


_NP2DT = {np.dtype(getattr(np, d.name)): d for d in Dtype}


class Coder(enum.IntEnum):  # entropy::Coder (entropy.hpp:11-14)
    arithmetic = 0
    rans = 1


class SvdBackend(enum.IntEnum):  # sthosvd::SvdBackend (sthosvd.hpp:48-52)
    automatic = 0
    gram = 1
    direct = 2


class _CParams(C.Structure):
    _fields_ = [
        ("has_target_re", C.c_int), ("target_re", C.c_double), ("has_target_sse", C.c_int),
        ("target_sse", C.c_double), ("rtmss", C.c_double), ("threads", C.c_int), ("method", C.c_int),
        ("has_storage_order", C.c_int), ("storage_order", C.c_uint64 * 8),
        ("has_mode_order", C.c_int), ("mode_order", C.c_uint64 * 8),
        ("coder", C.c_int), ("split_planes", C.c_int), ("simple_factor_weights", C.c_int),
        ("block_size", C.c_uint64), ("internal_float32", C.c_int), ("svd_backend", C.c_int),
    ]


class _CTimes(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("sthosvd_ms", "quantize_ms", "core_encode_ms", "factor_encode_ms",
                                          "serialize_ms", "total_ms")]


class _CResult(C.Structure):
    _fields_ = [
        ("container", C.POINTER(C.c_uint8)), ("container_size", C.c_uint64),
        ("truncation_sse", C.c_double), ("core_quantization_sse", C.c_double),
        ("factor_terms", C.c_double * 8), ("estimate_sse", C.c_double), ("norm_sq", C.c_double),
        ("target_sse", C.c_double), ("ranks", C.c_uint64 * 8), ("order", C.c_int), ("times", _CTimes),
        ("peak_alloc_estimate", C.c_uint64), ("original_bytes", C.c_uint64),
        ("ingest_precision_loss", C.c_int), ("core_last_plane", C.c_int), ("core_scale_exponent", C.c_int),
        ("uncertified_decisions", C.c_int), ("kernel_launches", C.c_uint64), ("rank_tie_modes", C.c_uint32),
    ]


def lib():
    """Load libtucomp_b200.so; raises TucompError if it was not built."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise TucompError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        L.tcb_last_error.restype = C.c_char_p
        L.tcb_kernel_launches.restype = C.c_uint64
        L.tcb_pinned_staging_allocs.restype = C.c_uint64
        _LIB = L
    return _LIB


def _check(rc: int):
    if rc != 0:
        raise TucompError(lib().tcb_last_error().decode())


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _take_bytes(ptr, n) -> bytes:
    out = C.string_at(ptr, n) if n else b""
    lib().tcb_free(C.cast(ptr, C.c_void_p))
    return out


def kernel_launches() -> int:
    return int(lib().tcb_kernel_launches())


def pinned_staging_allocs() -> int:
    return int(lib().tcb_pinned_staging_allocs())


# ---------------------------------------------------------------- pipeline API
@dataclass
class Params:
    """tucomp::pipeline::Params (pipeline.hpp:14-28)."""
    target_re: Optional[float] = None
    target_sse: Optional[float] = None
    rtmss: float = 0.5  # errormodel::kDefaultRtmss
    threads: int = 1
    method: int = 0  # vectorize::Method::lexicographic
    storage_order: Optional[Sequence[int]] = None
    mode_order: Optional[Sequence[int]] = None
    coder: int = Coder.arithmetic
    split_planes: bool = True
    simple_factor_weights: bool = False
    block_size: int = 0
    internal_float32: bool = False
    svd_backend: int = SvdBackend.automatic

    def to_c(self, d: int) -> _CParams:
        p = _CParams()
        p.has_target_re = int(self.target_re is not None)
        p.target_re = float(self.target_re or 0.0)
        p.has_target_sse = int(self.target_sse is not None)
        p.target_sse = float(self.target_sse or 0.0)
        p.rtmss = self.rtmss
        p.threads = self.threads
        p.method = int(self.method)
        if self.storage_order is not None:
            p.has_storage_order = 1
            for i, v in enumerate(self.storage_order):
                p.storage_order[i] = v
        if self.mode_order is not None:
            p.has_mode_order = 1
            for i, v in enumerate(self.mode_order):
                p.mode_order[i] = v
        p.coder = int(self.coder)
        p.split_planes = int(self.split_planes)
        p.simple_factor_weights = int(self.simple_factor_weights)
        p.block_size = self.block_size
        p.internal_float32 = int(self.internal_float32)
        p.svd_backend = int(self.svd_backend)
        return p


@dataclass
class SourceBuffer:
    """container::SourceBuffer (container.hpp:34-39)."""
    bytes: bytes
    dtype: Dtype
    shape: Sequence[int]
    skip_bytes: int = 0

    @staticmethod
    def from_array(a: np.ndarray) -> "SourceBuffer":
        a = np.ascontiguousarray(a)
        return SourceBuffer(a.tobytes(), _NP2DT[a.dtype], list(a.shape))


@dataclass
class PhaseTimes:
    sthosvd_ms: float = 0.0
    quantize_ms: float = 0.0
    core_encode_ms: float = 0.0
    factor_encode_ms: float = 0.0
    serialize_ms: float = 0.0
    total_ms: float = 0.0


@dataclass
class ErrorEstimate:
    truncation_sse: float = 0.0
    core_quantization_sse: float = 0.0
    factor_terms: list = field(default_factory=list)

    def total(self) -> float:
        t = self.truncation_sse + self.core_quantization_sse
        for f in self.factor_terms:
            t += f
        return t


@dataclass
class CompressResult:
    """tucomp::pipeline::CompressResult (pipeline.hpp:39-55)."""
    container: bytes
    estimate: ErrorEstimate
    norm_sq: float
    target_sse: float
    ranks: list
    times: PhaseTimes
    peak_alloc_estimate: int
    original_bytes: int
    ingest_precision_loss: bool
    core_last_plane: int = 63
    core_scale_exponent: int = 0
    uncertified_decisions: int = 0
    kernel_launches: int = 0
    rank_tie_modes: int = 0

    def compression_factor(self) -> float:
        return 0.0 if not self.container else self.original_bytes / len(self.container)


def _result(r: _CResult) -> CompressResult:
    d = r.order
    t = r.times
    return CompressResult(
        container=_take_bytes(r.container, r.container_size),
        estimate=ErrorEstimate(r.truncation_sse, r.core_quantization_sse, [r.factor_terms[i] for i in range(d)]),
        norm_sq=r.norm_sq, target_sse=r.target_sse, ranks=[int(r.ranks[i]) for i in range(d)],
        times=PhaseTimes(t.sthosvd_ms, t.quantize_ms, t.core_encode_ms, t.factor_encode_ms, t.serialize_ms,
                         t.total_ms),
        peak_alloc_estimate=r.peak_alloc_estimate, original_bytes=r.original_bytes,
        ingest_precision_loss=bool(r.ingest_precision_loss), core_last_plane=r.core_last_plane,
        core_scale_exponent=r.core_scale_exponent, uncertified_decisions=r.uncertified_decisions,
        kernel_launches=int(r.kernel_launches), rank_tie_modes=int(r.rank_tie_modes))


def compress(src: SourceBuffer, params: Params) -> CompressResult:
    """tucomp::pipeline::compress (pipeline.cpp:240-252) on the B200."""
    return _result(compress_raw(src, params))


def compress_raw(src: SourceBuffer, params: Params) -> "_CResult":
    """tcb_compress itself (the C ABI a reference-side binding calls): the
    container is in host memory when this returns; free it with
    free_raw() or turn the result into a CompressResult with _result()."""
    shape = np.asarray(list(src.shape), np.uint64)
    buf = np.frombuffer(src.bytes, np.uint8) if len(src.bytes) else np.zeros(1, np.uint8)
    res = _CResult()
    _check(lib().tcb_compress(_p(buf), C.c_uint64(len(src.bytes)), int(src.dtype), _p(shape), len(shape),
                              C.c_uint64(src.skip_bytes), C.byref(params.to_c(len(shape))), C.byref(res)))
    return res


def free_raw(res: "_CResult") -> None:
    lib().tcb_free(C.cast(res.container, C.c_void_p))


def compress_device(ptr: int, nbytes: int, dtype: Dtype, shape: Sequence[int], params: Params) -> CompressResult:
    """Same as compress() with the element bytes already resident in device memory (e.g. a torch tensor)."""
    return _result(compress_device_raw(ptr, nbytes, dtype, shape, params))


def compress_device_raw(ptr: int, nbytes: int, dtype: Dtype, shape: Sequence[int], params: Params) -> "_CResult":
    """tcb_compress_device itself: the container is in (pinned) host memory when this
    returns; _result() turns it into a CompressResult (copying it into a Python bytes)."""
    sh = np.asarray(list(shape), np.uint64)
    res = _CResult()
    _check(lib().tcb_compress_device(C.c_void_p(ptr), C.c_uint64(nbytes), int(dtype), _p(sh), len(sh),
                                     C.byref(params.to_c(len(sh))), C.byref(res)))
    return res


def measure_error(src: SourceBuffer, container: bytes, internal_float32: bool = False) -> float:
    """The CLI's measure_error (tools/tucomp_main.cpp:121-135) on the device:
    sse_between(ingest(src), decompress_tensor(container)) (tensor.cpp:147-164)."""
    shape = np.asarray(list(src.shape), np.uint64)
    buf = np.frombuffer(src.bytes, np.uint8) if len(src.bytes) else np.zeros(1, np.uint8)
    cb = np.frombuffer(container, np.uint8) if len(container) else np.zeros(1, np.uint8)
    sse = C.c_double()
    _check(lib().tcb_measure_error(_p(buf), C.c_uint64(len(src.bytes)), int(src.dtype), _p(shape), len(shape),
                                   C.c_uint64(src.skip_bytes), int(bool(internal_float32)), _p(cb),
                                   C.c_uint64(len(container)), C.byref(sse)))
    return float(sse.value)


class _CDecompress(C.Structure):  # tcb_decompress_result
    _fields_ = [("bytes", C.POINTER(C.c_uint8)), ("nbytes", C.c_uint64), ("dtype", C.c_int), ("d", C.c_int),
                ("shape", C.c_uint64 * 8), ("total_ms", C.c_double)]


class _LibBuffer:
    """A library-owned result buffer (tcb_free when the last view goes): numpy
    views made from it keep it alive through __array_interface__."""

    def __init__(self, ptr, n):
        self.ptr = C.cast(ptr, C.c_void_p)
        self.n = int(n)
        self.__array_interface__ = {"shape": (self.n,), "typestr": "|u1", "version": 3,
                                    "data": (self.ptr.value or 0, True)}

    @property
    def array(self) -> np.ndarray:
        return np.asarray(self) if self.n else np.zeros(0, np.uint8)

    def __del__(self):
        if self.ptr:
            lib().tcb_free(self.ptr)
            self.ptr = None


_NP_OF = {0: np.int8, 1: np.uint8, 2: np.int16, 3: np.uint16, 4: np.int32, 5: np.uint32, 6: np.int64,
          7: np.uint64, 8: np.float32, 9: np.float64}


class DecompressResult:  # pipeline::DecompressResult (pipeline.hpp:59-64)
    """Decompressed source-dtype bytes; `to_array()` views them without a copy
    (the buffer lives in the library's pinned pool until this object goes)."""

    def __init__(self, buf: "_LibBuffer", dtype: "Dtype", shape: tuple, total_ms: float):
        self._buf = buf
        self.dtype = dtype
        self.shape = shape
        self.total_ms = total_ms

    @property
    def bytes(self) -> bytes:
        return self._buf.array.tobytes()

    def to_array(self) -> np.ndarray:
        a = self._buf.array.view(_NP_OF[int(self.dtype)]).reshape(self.shape)
        a.flags.writeable = False
        return a


def decompress(container: bytes, threads: int = 1) -> DecompressResult:
    """tucomp::pipeline::decompress (pipeline.cpp:266-283) on the B200: decode,
    reconstruct and emit the source dtype's bytes (container.cpp:98-140)."""
    buf = np.frombuffer(container, np.uint8) if len(container) else np.zeros(1, np.uint8)
    r = _CDecompress()
    _check(lib().tcb_decompress(_p(buf), C.c_uint64(len(container)), int(threads), C.byref(r)))
    return DecompressResult(_LibBuffer(r.bytes, r.nbytes), Dtype(r.dtype),
                            tuple(int(r.shape[i]) for i in range(r.d)), float(r.total_ms))


def decompress_device(container: bytes, device_ptr: int, capacity: int):
    """pipeline::decompress into device memory (B200 extension): the emitted
    source-dtype bytes land at `device_ptr`; returns (dtype, shape, total_ms)."""
    buf = np.frombuffer(container, np.uint8) if len(container) else np.zeros(1, np.uint8)
    r = _CDecompress()
    _check(lib().tcb_decompress_device(_p(buf), C.c_uint64(len(container)), C.c_void_p(device_ptr),
                                       C.c_uint64(capacity), C.byref(r)))
    return Dtype(r.dtype), tuple(int(r.shape[i]) for i in range(r.d)), float(r.total_ms)


def decompress_tensor(container: bytes) -> np.ndarray:
    """tucomp::pipeline::decompress_tensor<double> (pipeline.hpp:70-71) on the B200."""
    buf = np.frombuffer(container, np.uint8) if len(container) else np.zeros(1, np.uint8)
    ptr = C.POINTER(C.c_double)()
    cnt, d = C.c_uint64(), C.c_int()
    shape = (C.c_uint64 * 8)()
    _check(lib().tcb_decompress_tensor_f64(_p(buf), C.c_uint64(len(container)), C.byref(ptr), C.byref(cnt), shape,
                                           C.byref(d)))
    n = int(cnt.value)
    out = np.ctypeslib.as_array(ptr, shape=(n,)).copy() if n else np.zeros(0)
    lib().tcb_free(C.cast(ptr, C.c_void_p))
    return out.reshape(tuple(int(shape[i]) for i in range(d.value)))


class _CHeader(C.Structure):  # tcb_container_header
    _fields_ = [(n, C.c_int) for n in ("version", "source_dtype", "internal_float32", "d", "coder", "method",
                                       "zero_flag", "split_planes", "simple_weights")] + \
               [(n, C.c_uint64 * 8) for n in ("mode_sizes", "ranks", "processing_order", "storage_order")] + \
               [("core_scale_exponent", C.c_int), ("block_size", C.c_uint64)] + \
               [(n, C.c_double) for n in ("rtmss", "target_sse", "norm_sq", "truncation_sse", "core_quant_sse",
                                          "estimate_sse")]


@dataclass
class Header:  # container::Header (container.hpp:59-82); orders 0-based
    version: int
    source_dtype: Dtype
    internal_float32: bool
    mode_sizes: tuple
    ranks: tuple
    processing_order: tuple
    storage_order: tuple
    method: int
    coder: int
    zero_flag: bool
    split_planes: bool
    simple_weights: bool
    core_scale_exponent: int
    block_size: int
    rtmss: float
    target_sse: float
    norm_sq: float
    truncation_sse: float
    core_quant_sse: float
    estimate_sse: float

    def order(self) -> int:
        return len(self.mode_sizes)

    def element_count(self) -> int:
        return int(np.prod(self.mode_sizes, dtype=object))


def read_container(container: bytes) -> Header:
    """container::read_container (container.cpp:338-420): the header, after every
    header and section-structure check.  Host only (no device work)."""
    buf = np.frombuffer(container, np.uint8) if len(container) else np.zeros(1, np.uint8)
    h = _CHeader()
    _check(lib().tcb_read_container_header(_p(buf), C.c_uint64(len(container)), C.byref(h)))
    d = h.d
    t = lambda a: tuple(int(a[i]) for i in range(d))  # noqa: E731
    return Header(h.version, Dtype(h.source_dtype), bool(h.internal_float32), t(h.mode_sizes), t(h.ranks),
                  t(h.processing_order), t(h.storage_order), h.method, h.coder, bool(h.zero_flag),
                  bool(h.split_planes), bool(h.simple_weights), h.core_scale_exponent, int(h.block_size), h.rtmss,
                  h.target_sse, h.norm_sq, h.truncation_sse, h.core_quant_sse, h.estimate_sse)


# ---------------------------------------------------------------- lower-level ops
def sthosvd(a: np.ndarray, sse_target: float, order=None, backend=0) -> dict:
    """sthosvd::compress<double> (sthosvd.hpp:66-68) on the device."""
    a = np.ascontiguousarray(a, np.float64)
    d = a.ndim
    shape = np.asarray(a.shape, np.uint64)
    core = np.zeros(a.size)
    cs = (C.c_uint64 * d)()
    facs = [np.zeros(n * n) for n in a.shape]
    fptr = (C.c_void_p * d)(*[f.ctypes.data for f in facs])
    ranks = (C.c_uint64 * d)()
    trunc = (C.c_double * d)()
    ordo = (C.c_uint64 * d)()
    oarr = np.asarray(order, np.uint64) if order is not None else None
    _check(lib().tcb_sthosvd_f64(_p(a), _p(shape), d, C.c_double(sse_target),
                                 _p(oarr) if oarr is not None else None, backend, _p(core), cs, fptr, ranks, trunc,
                                 ordo))
    core_shape = [int(cs[i]) for i in range(d)]
    rk = [int(ranks[i]) for i in range(d)]
    return dict(core=core[:int(np.prod(core_shape))].reshape(core_shape), ranks=rk,
                trunc=[trunc[i] for i in range(d)], order=[int(ordo[i]) for i in range(d)],
                factors=[facs[i][:a.shape[i] * rk[i]].reshape(a.shape[i], rk[i]) for i in range(d)])


def gram(b: np.ndarray) -> np.ndarray:
    b = np.ascontiguousarray(b, np.float64)
    g = np.zeros((b.shape[0], b.shape[0]))
    _check(lib().tcb_gram_f64(_p(b), C.c_uint64(b.shape[0]), C.c_uint64(b.shape[1]), _p(g)))
    return g


def ttm(b: np.ndarray, u: np.ndarray) -> np.ndarray:
    b = np.ascontiguousarray(b, np.float64)
    u = np.ascontiguousarray(u, np.float64)
    out = np.zeros((b.shape[1], u.shape[1]))
    _check(lib().tcb_ttm_f64(_p(b), C.c_uint64(b.shape[0]), C.c_uint64(b.shape[1]), _p(u), C.c_uint64(u.shape[1]),
                             _p(out)))
    return out


def eig(g: np.ndarray, r: int):
    """Descending eigenvalues and the top-r sign-fixed eigenvectors of a symmetric matrix."""
    g = np.ascontiguousarray(g, np.float64)
    n = g.shape[0]
    ev = np.zeros(n)
    u = np.zeros((n, max(r, 1)))
    _check(lib().tcb_eig_f64(_p(g), C.c_uint64(n), C.c_uint64(r), _p(ev), _p(u)))
    return ev, u[:, :r]


def quantize(core: np.ndarray):
    core = np.ascontiguousarray(core, np.float64)
    shape = np.asarray(core.shape, np.uint64)
    mag = np.zeros(core.size, np.uint64)
    neg = np.zeros(core.size, np.uint8)
    k = C.c_int()
    zero = C.c_int()
    sn = np.zeros(int(sum(core.shape)))
    _check(lib().tcb_quantize_f64(_p(core), _p(shape), core.ndim, _p(mag), _p(neg), C.byref(k), C.byref(zero),
                                  _p(sn)))
    parts, o = [], 0
    for e in core.shape:
        parts.append(sn[o:o + e].copy())
        o += e
    return mag, neg, k.value, bool(zero.value), parts


def encode(mag, neg, target_int, coder=0, block_size=0, split=True, fixed_plane=-1):
    """corecodec::Encoder plan+finalize; returns (stream section, last_plane, achieved_sse_int, decoded, uncertified)."""
    mag = np.ascontiguousarray(mag, np.uint64)
    neg = np.ascontiguousarray(neg, np.uint8)
    n = mag.size
    out = C.POINTER(C.c_uint8)()
    ln = C.c_uint64()
    lp = C.c_int()
    ach = C.c_double()
    unc = C.c_int()
    dec = np.zeros(max(n, 1), np.uint64)
    _check(lib().tcb_encode(_p(mag) if n else None, _p(neg) if n else None, C.c_uint64(n), C.c_double(target_int),
                            coder, C.c_uint64(block_size), int(split), fixed_plane, C.byref(out), C.byref(ln),
                            C.byref(lp), C.byref(ach), _p(dec), C.byref(unc)))
    return _take_bytes(out, ln.value), lp.value, ach.value, dec[:n], unc.value


EX_LEAD, EX_TRAIL, EX_BOTH, EX_SQ, EX_RECAL, EX_DIFF = range(6)


def exact_sums(mag, segs, kinds, dec=None, reference=False):
    """The encoder's serial double sums, bit-exact (tcb_exact_sums).  segs: list of
    (lo, hi, backward, s0, need) with need=inf for a plain sum; kinds: list of
    (term, plane).  Returns (sums, c0, c1, crossed), each of shape (len(kinds), len(segs))."""
    mag = np.ascontiguousarray(mag, np.uint64)
    n = mag.size
    d = None if dec is None else np.ascontiguousarray(dec, np.uint64)
    g = len(segs)
    lo = np.array([x[0] for x in segs], np.uint64)
    hi = np.array([x[1] for x in segs], np.uint64)
    bw = np.array([int(x[2]) for x in segs], np.int32)
    s0 = np.array([float(x[3]) for x in segs], np.float64)
    nd = np.array([float(x[4]) for x in segs], np.float64)
    kt = np.array([k[0] for k in kinds], np.int32)
    kp = np.array([k[1] for k in kinds], np.int32)
    nj = max(1, g * len(kinds))
    sums = np.zeros(nj, np.float64)
    c0 = np.zeros(nj, np.uint64)
    c1 = np.zeros(nj, np.uint64)
    cr = np.zeros(nj, np.int32)
    _check(lib().tcb_exact_sums(_p(mag) if n else None, _p(d) if d is not None else None, C.c_uint64(n), _p(lo), _p(hi),
                                _p(bw), _p(s0), _p(nd), g, _p(kt), _p(kp), len(kinds), int(reference), _p(sums),
                                _p(c0), _p(c1), _p(cr)))
    shp = (len(kinds), g)
    nj = g * len(kinds)
    return sums[:nj].reshape(shp), c0[:nj].reshape(shp), c1[:nj].reshape(shp), cr[:nj].reshape(shp)


def plane_stats(mag, block, p_top, np_):
    """build_block's exact per-block statistics of planes p_top..p_top-np_+1 (tcb_exact_plane_stats);
    same layout as exact_sums over kinds [(lead, p), (trail, p) for p descending] and the block segments."""
    mag = np.ascontiguousarray(mag, np.uint64)
    n = mag.size
    nb = (n + block - 1) // block
    nj = max(1, 2 * np_ * nb)
    sums = np.zeros(nj, np.float64)
    c0 = np.zeros(nj, np.uint64)
    c1 = np.zeros(nj, np.uint64)
    cr = np.zeros(nj, np.int32)
    _check(lib().tcb_exact_plane_stats(_p(mag) if n else None, C.c_uint64(n), C.c_uint64(block), int(p_top), int(np_),
                                       _p(sums), _p(c0), _p(c1), _p(cr)))
    shp = (2 * np_, nb)
    k = 2 * np_ * nb
    return sums[:k].reshape(shp), c0[:k].reshape(shp), c1[:k].reshape(shp), cr[:k].reshape(shp)


def encode_symbols(coder, syms) -> bytes:
    s = np.ascontiguousarray(syms, np.uint64)
    out = C.POINTER(C.c_uint8)()
    ln = C.c_uint64()
    _check(lib().tcb_encode_symbols(coder, _p(s) if s.size else None, C.c_uint64(s.size), C.byref(out),
                                    C.byref(ln)))
    return _take_bytes(out, ln.value)


def encode_factor(u, dead, slice_norms, coder=0, simple=False, core_step_log2=0, term_cap=0.0) -> dict:
    u = np.ascontiguousarray(u, np.float64)
    n, r = u.shape
    dead = np.ascontiguousarray(dead, np.uint8)
    sn = np.ascontiguousarray(slice_norms, np.float64)
    out = C.POINTER(C.c_uint8)()
    ln = C.c_uint64()
    k = C.c_int()
    cnt = C.c_uint64()
    flips = np.zeros(max(r, 1), np.int8)
    term = C.c_double()
    plane = C.c_int()
    _check(lib().tcb_encode_factor_f64(_p(u), C.c_uint64(n), C.c_uint64(r), _p(dead), _p(sn), coder, int(simple),
                                       core_step_log2, C.c_double(term_cap), C.byref(out), C.byref(ln), C.byref(k),
                                       C.byref(cnt), _p(flips), C.byref(term), C.byref(plane)))
    return dict(stream=_take_bytes(out, ln.value), k=k.value, count=cnt.value, flips=flips[:r], term=term.value,
                plane=plane.value)


EXPORTED = ("tcb_compress", "tcb_compress_device", "tcb_decompress", "tcb_decompress_tensor_f64", "tcb_decompress_device", "tcb_read_container_header",
            "tcb_nccl_unique_id", "tcb_nccl_comm_init", "tcb_nccl_comm_destroy", "tcb_compress_sharded_device",
            "tcb_compress_sharded_host", "tcb_dev_encode_tucker_sharded", "tcb_measure_error",
            "tcb_default_params", "tcb_free", "tcb_last_error",
            "tcb_kernel_launches", "tcb_pinned_staging_allocs", "tcb_sthosvd_f64", "tcb_gram_f64", "tcb_ttm_f64", "tcb_eig_f64",
            "tcb_quantize_f64", "tcb_encode", "tcb_exact_sums", "tcb_exact_plane_stats", "tcb_encode_symbols", "tcb_encode_factor_f64")
