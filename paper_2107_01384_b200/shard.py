"""Sharded multi-GPU ST-HOSVD mode loop (reference
sthosvd.cpp:114-171 run across ranks).

The tensor is partitioned along the LAST processed mode p[d-1]: rank k holds a
contiguous slab of that mode.  Thanks to the circular shift (the TTM output of
step s is the next step's tensor, sthosvd.cpp:158-166) the sharded mode moves
one axis to the left per step and is never the contracted (row) axis before
the last step, so for steps 0..d-2:

    local Gram of the column shard -> all_reduce(SUM) -> replicated eigensolve
    + rank rule (bitwise identical on every rank, deterministic kernels on an
    identical Gram) -> shard-local TTM, no data exchange.

Before the last step the (small) tensor is all-gathered along its leading axis
and the last step runs replicated; rank 0 encodes the core.  If a middle step
hits the rows > cols branch (sthosvd.cpp:75-76) its tensor is gathered along
the sharded axis, the step runs replicated and every rank keeps its slab.

`ops` supplies the per-rank compute: DeviceOps (B200 kernels through the C
ABI, NCCL collectives) or, in the CPU tests, a numpy implementation.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import Params, TucompError, _check, _result, _CResult, lib


def shard_bounds(extent: int, world: int, rank: int):
    """Contiguous split of one mode: first `extent % world` ranks get one more."""
    base, extra = divmod(extent, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def stable_ascending(shape):
    return sorted(range(len(shape)), key=lambda i: (shape[i], i))


class DeviceOps:
    """B200 kernels on torch CUDA float64 tensors (device pointers into the C ABI)."""

    @staticmethod
    def _p(t):
        return C.c_void_p(t.data_ptr())

    def sumsq(self, x):
        torch.cuda.synchronize()
        out, fin = C.c_double(), C.c_int()
        _check(lib().tcb_dev_sumsq(self._p(x), C.c_uint64(x.numel()), C.byref(out), C.byref(fin)))
        return out.value, bool(fin.value)

    def permute(self, x, perm):
        shape = np.asarray(x.shape, np.uint64)
        pm = np.asarray(perm, np.uint64)
        out = torch.empty([x.shape[i] for i in perm], dtype=x.dtype, device=x.device)
        torch.cuda.synchronize()
        _check(lib().tcb_dev_permute(self._p(x), self._p(out), shape.ctypes.data_as(C.c_void_p),
                                     pm.ctypes.data_as(C.c_void_p), x.dim()))
        return out

    def gram(self, b2):
        rows, cols = b2.shape
        g = torch.empty((rows, rows), dtype=torch.float64, device=b2.device)
        torch.cuda.synchronize()
        _check(lib().tcb_dev_gram(self._p(b2), C.c_uint64(rows), C.c_uint64(cols), self._p(g)))
        return g

    def gram_ozaki(self, b2):
        rows, cols = b2.shape
        g = torch.empty((rows, rows), dtype=torch.float64, device=b2.device)
        torch.cuda.synchronize()
        _check(lib().tcb_dev_gram_ozaki(self._p(b2), C.c_uint64(rows), C.c_uint64(cols), self._p(g)))
        return g

    def ttm_ozaki(self, b2, u):
        rows, cols = b2.shape
        r = u.shape[1]
        out = torch.empty((cols, r), dtype=torch.float64, device=b2.device)
        torch.cuda.synchronize()
        _check(lib().tcb_dev_ttm_ozaki(self._p(b2), C.c_uint64(rows), C.c_uint64(cols), self._p(u.contiguous()),
                                       C.c_uint64(r), self._p(out)))
        return out

    def factor_from_gram(self, g, budget):
        n = g.shape[0]
        u = torch.empty(n * n, dtype=torch.float64, device=g.device)
        r, disc = C.c_uint64(), C.c_double()
        torch.cuda.synchronize()
        _check(lib().tcb_dev_factor_from_gram(self._p(g), C.c_uint64(n), C.c_double(budget), self._p(u),
                                              C.byref(r), C.byref(disc)))
        return u[: n * r.value].view(n, r.value), r.value, disc.value

    def ttm(self, b2, u):
        rows, cols = b2.shape
        r = u.shape[1]
        out = torch.empty((cols, r), dtype=torch.float64, device=b2.device)
        torch.cuda.synchronize()
        _check(lib().tcb_dev_ttm(self._p(b2), C.c_uint64(rows), C.c_uint64(cols), self._p(u.contiguous()),
                                 C.c_uint64(r), self._p(out)))
        return out

    def mode_step(self, b2, budget, backend):
        rows, cols = b2.shape
        u = torch.empty(rows * rows, dtype=torch.float64, device=b2.device)
        nx = torch.empty(cols * rows, dtype=torch.float64, device=b2.device)
        r, disc = C.c_uint64(), C.c_double()
        torch.cuda.synchronize()
        _check(lib().tcb_dev_mode_step(self._p(b2), C.c_uint64(rows), C.c_uint64(cols), C.c_double(budget),
                                       int(backend), self._p(u), self._p(nx), C.byref(r), C.byref(disc)))
        return u[: rows * r.value].view(rows, r.value), nx[: cols * r.value].view(cols, r.value), r.value, disc.value

    def encode(self, core, factors, n, r, order, trunc, dtype, norm_sq, target, params: Params):
        d = len(n)
        arr = lambda v, t: np.asarray(v, t)  # noqa: E731
        na, ra, oa, ta = arr(n, np.uint64), arr(r, np.uint64), arr(order, np.uint64), arr(trunc, np.float64)
        fptr = (C.c_void_p * d)(*[f.data_ptr() for f in factors])
        res = _CResult()
        torch.cuda.synchronize()
        _check(lib().tcb_dev_encode_tucker(self._p(core), fptr, na.ctypes.data_as(C.c_void_p),
                                           ra.ctypes.data_as(C.c_void_p), oa.ctypes.data_as(C.c_void_p),
                                           ta.ctypes.data_as(C.c_void_p), d, int(dtype), C.c_double(norm_sq),
                                           C.c_double(target), C.byref(params.to_c(d)), C.byref(res)))
        return _result(res)


@dataclass
class ShardedTucker:
    core: object            # processing-order core (replicated)
    factors: list           # by original mode, n_i x r_i
    ranks: list
    order: list
    trunc: list
    norm_sq: float


def _all_gather_cat(t, axis, group, world):
    """Concatenate every rank's tensor along `axis` (extents may differ per rank)."""
    if world == 1:
        return t
    sizes = [torch.zeros(1, dtype=torch.int64, device=t.device) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([t.shape[axis]], dtype=torch.int64, device=t.device), group=group)
    sizes = [int(s.item()) for s in sizes]
    mx = max(sizes)
    pad_shape = list(t.shape)
    pad_shape[axis] = mx
    padded = torch.zeros(pad_shape, dtype=t.dtype, device=t.device)
    padded.narrow(axis, 0, t.shape[axis]).copy_(t)
    bufs = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(bufs, padded.contiguous(), group=group)
    return torch.cat([b.narrow(axis, 0, s) for b, s in zip(bufs, sizes)], dim=axis).contiguous()


def _global_stats(x_local, ops, group, world):
    """(||x||^2 over all ranks, every value finite on every rank) in one pass per rank."""
    ssq, finite = ops.sumsq(x_local)
    stats = torch.tensor([ssq, 0.0 if finite else 1.0], dtype=torch.float64, device=x_local.device)
    if world > 1:
        dist.all_reduce(stats, group=group)
    return float(stats[0].item()), stats[1].item() == 0.0


def sthosvd_sharded(x_local, shape, target, ops, order=None, backend=0, group=None, stats=None):
    """ST-HOSVD over ranks; `x_local` is this rank's slab of mode order[-1]
    (original axis order).  `stats` = (norm^2, all finite) when the caller
    already scanned the input.  Returns the replicated factorization."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    d = len(shape)
    p = list(order) if order is not None else stable_ascending(shape)
    norm_sq, finite = stats if stats is not None else _global_stats(x_local, ops, group, world)
    if target < 0:
        raise TucompError("sthosvd: negative SSE target")
    if not finite:
        raise TucompError("sthosvd: input contains non-finite values")
    # identity processing order: mode 0 reads the slab in place (tensor.cpp:105-144 is a no-op then)
    xl = x_local.contiguous() if p == list(range(d)) else ops.permute(x_local, p)
    cur = list(xl.shape)
    sh_axis = d - 1  # position of the sharded mode in `cur`
    remaining = float(target)
    factors, ranks, trunc = [None] * d, [0] * d, [0.0] * d
    for step in range(d):
        budget = remaining / float(d - step)
        rows = cur[0]
        if sh_axis == 0 or step == d - 1:
            full = _all_gather_cat(xl.view(cur), 0, group, world) if sh_axis == 0 else xl.view(cur)
            fc = list(full.shape)
            u, nx, r, disc = ops.mode_step(full.view(fc[0], -1), budget, backend)
            xl = nx
            cur = fc[1:] + [r]
            sh_axis = -1  # replicated from here on
        else:
            cols_local = int(np.prod(cur[1:]))
            cols_t = torch.tensor([float(cols_local)], dtype=torch.float64, device=xl.device)
            if world > 1:
                dist.all_reduce(cols_t, group=group)
            cols_global = int(cols_t.item())
            via_gram = backend == 1 or (backend == 0 and rows <= cols_global)
            if via_gram:
                g = ops.gram(xl.view(rows, cols_local))
                if world > 1:
                    dist.all_reduce(g, group=group)
                u, r, disc = ops.factor_from_gram(g, budget)
                xl = ops.ttm(xl.view(rows, cols_local), u)
                cur = cur[1:] + [r]
                sh_axis -= 1
            else:  # thin-SVD branch: gather along the sharded axis, step replicated, keep my slab
                full = _all_gather_cat(xl.view(cur), sh_axis, group, world)
                fc = list(full.shape)
                u, nx, r, disc = ops.mode_step(full.view(fc[0], -1), budget, backend)
                nfull = nx.view(fc[1:] + [r])
                sh_axis -= 1
                lo, hi = shard_bounds(fc[sh_axis + 1], world, rank)
                xl = nfull.narrow(sh_axis, lo, hi - lo).contiguous()
                cur = list(xl.shape)
        remaining = max(0.0, remaining - disc)
        trunc[p[step]] = disc
        factors[p[step]] = u
        ranks[p[step]] = r
    return ShardedTucker(core=xl.view(cur), factors=factors, ranks=ranks, order=p, trunc=trunc,
                         norm_sq=norm_sq)


_COMMS = {}


def _nccl_comm(group, world, rank, device):
    """The library's own NCCL communicator for `group` (created once): rank 0's
    unique id travels through torch.distributed."""
    key = (id(group), world, rank)
    if key in _COMMS:
        return _COMMS[key]
    uid = (C.c_uint8 * 128)()
    if rank == 0:
        _check(lib().tcb_nccl_unique_id(uid))
    backend = dist.get_backend(group) if dist.is_initialized() else "gloo"
    t = torch.tensor(list(bytes(uid)), dtype=torch.uint8,
                     device=device if backend == "nccl" else "cpu")
    if world > 1:
        dist.broadcast(t, src=0, group=group)
    uid = (C.c_uint8 * 128)(*t.cpu().tolist())
    comm = C.c_void_p()
    _check(lib().tcb_nccl_comm_init(uid, int(world), int(rank), C.byref(comm)))
    _COMMS[key] = comm
    return comm


# ---------------------------------------------------------------- host-memory collectives
_ALLREDUCE_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_uint64)
_ALLGATHER_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64)


class _CHostColl(C.Structure):  # tcb_host_collectives
    _fields_ = [("ctx", C.c_void_p), ("allreduce_sum_f64", _ALLREDUCE_CB), ("allgather", _ALLGATHER_CB)]


class HostCollectives:
    """The library's collectives carried by torch.distributed on host tensors
    (any backend with CPU support, e.g. gloo): the sharded C++ pipeline then
    runs without NCCL -- several ranks may even share one GPU, since no kernel
    of one rank waits on another rank."""

    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1

        def allreduce(ctx, buf, n):
            try:
                t = torch.from_numpy(np.ctypeslib.as_array(buf, shape=(int(n),)))
                dist.all_reduce(t, group=self.group)
                return 0
            except Exception:  # noqa: BLE001 -- reported to the library as a failure
                return 1

        def allgather(ctx, send, recv, nbytes):
            try:
                nb = int(nbytes)
                src = torch.from_numpy(np.ctypeslib.as_array((C.c_uint8 * nb).from_address(send))) if nb else \
                    torch.zeros(0, dtype=torch.uint8)
                out = [torch.empty(nb, dtype=torch.uint8) for _ in range(self.world)]
                dist.all_gather(out, src.clone(), group=self.group)
                if nb:
                    dst = np.ctypeslib.as_array((C.c_uint8 * (nb * self.world)).from_address(recv))
                    for r, t in enumerate(out):
                        dst[r * nb:(r + 1) * nb] = t.numpy()
                return 0
            except Exception:  # noqa: BLE001
                return 1

        self._ar = _ALLREDUCE_CB(allreduce)  # keep the thunks alive
        self._ag = _ALLGATHER_CB(allgather)
        self.c = _CHostColl(None, self._ar, self._ag)


def compress_sharded_host(x_local, shape, dtype, params: Params, group=None):
    """The library's sharded compress with host collectives (HostCollectives):
    rank 0 returns the CompressResult, the other ranks None."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    p = list(params.mode_order) if params.mode_order is not None else stable_ascending(shape)
    lo, hi = shard_bounds(shape[p[-1]], world, rank)
    hc = HostCollectives(group)
    sh = np.asarray(list(shape), np.uint64)
    res = _CResult()
    with torch.cuda.device(x_local.device):
        torch.cuda.synchronize()
        _check(lib().tcb_compress_sharded_host(C.byref(hc.c), int(world), int(rank), C.c_void_p(x_local.data_ptr()),
                                               C.c_uint64(x_local.numel() * x_local.element_size()), int(dtype),
                                               sh.ctypes.data_as(C.c_void_p), len(shape), C.c_uint64(hi - lo),
                                               C.byref(params.to_c(len(shape))), C.byref(res)))
    out = _result(res)
    return out if rank == 0 else None


def encode_tucker_sharded(core, factors, n, r, order, trunc, dtype, norm_sq, target, params: Params, group=None,
                          host=True):
    """Encode an existing device Tucker factorization with the core's blocks split
    over the ranks (every rank holds the whole factorization); rank 0 returns the
    CompressResult."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    d = len(n)
    arr = lambda v, t: np.asarray(v, t)  # noqa: E731
    na, ra, oa, ta = arr(n, np.uint64), arr(r, np.uint64), arr(order, np.uint64), arr(trunc, np.float64)
    fptr = (C.c_void_p * d)(*[f.data_ptr() for f in factors])
    res = _CResult()
    hc = HostCollectives(group) if host else None
    comm = None if host else _nccl_comm(group, world, rank, core.device)
    torch.cuda.synchronize()
    _check(lib().tcb_dev_encode_tucker_sharded(comm, C.byref(hc.c) if hc else None, int(world), int(rank),
                                               C.c_void_p(core.data_ptr()), fptr, na.ctypes.data_as(C.c_void_p),
                                               ra.ctypes.data_as(C.c_void_p), oa.ctypes.data_as(C.c_void_p),
                                               ta.ctypes.data_as(C.c_void_p), d, int(dtype), C.c_double(norm_sq),
                                               C.c_double(target), C.byref(params.to_c(d)), C.byref(res)))
    out = _result(res)
    return out if rank == 0 else None


def _compress_sharded_cpp(x_local, shape, dtype, params: Params, group, world, rank):
    """The whole sharded compress in the library (mode loop, NCCL collectives,
    encode on rank 0): the single-GPU pipeline's kernels and concurrency."""
    p = list(params.mode_order) if params.mode_order is not None else stable_ascending(shape)
    last = p[-1]
    lo, hi = shard_bounds(shape[last], world, rank)
    with torch.cuda.device(x_local.device):  # the library works on the calling thread's device
        return _compress_sharded_cpp_on(x_local, shape, dtype, params, group, world, rank, hi - lo)


def _compress_sharded_cpp_on(x_local, shape, dtype, params, group, world, rank, local_extent):
    comm = _nccl_comm(group, world, rank, x_local.device)
    sh = np.asarray(list(shape), np.uint64)
    res = _CResult()
    torch.cuda.synchronize()
    _check(lib().tcb_compress_sharded_device(comm, int(world), int(rank), C.c_void_p(x_local.data_ptr()),
                                             C.c_uint64(x_local.numel() * x_local.element_size()), int(dtype),
                                             sh.ctypes.data_as(C.c_void_p), len(shape), C.c_uint64(local_extent),
                                             C.byref(params.to_c(len(shape))), C.byref(res)))
    out = _result(res)
    return out if rank == 0 else None


def compress_sharded(x_local, shape, dtype, params: Params, ops=None, group=None):
    """pipeline::compress across the ranks of `group`; rank 0 returns the
    CompressResult (container bytes), the other ranks return None.  On CUDA
    tensors with equal slabs the library runs the whole sharded pipeline (NCCL
    inside); otherwise the per-stage path below."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if ops is None and isinstance(x_local, torch.Tensor) and x_local.is_cuda and x_local.is_contiguous():
        p = list(params.mode_order) if params.mode_order is not None else stable_ascending(shape)
        if shape[p[-1]] % world == 0:
            try:
                return _compress_sharded_cpp(x_local, shape, dtype, params, group, world, rank)
            except TucompError as e:
                if "off the Gram route" not in str(e):
                    raise
    ops = ops or DeviceOps()
    if params.target_re is not None and params.target_sse is not None:
        raise TucompError("compress: relative-error and SSE targets are mutually exclusive")
    if params.target_re is None and params.target_sse is None:
        raise TucompError("compress: no error target given")
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    norm_sq, finite = _global_stats(x_local, ops, group, world)
    target = params.target_re ** 2 * norm_sq if params.target_re is not None else params.target_sse
    if target < 0:
        raise TucompError("budget: negative SSE target")
    if not 0.0 <= params.rtmss <= 1.0:
        raise TucompError("budget: rtmss outside [0, 1]")
    f = sthosvd_sharded(x_local, shape, params.rtmss * target, ops, params.mode_order, params.svd_backend, group,
                        stats=(norm_sq, finite))
    if rank != 0:
        return None
    return ops.encode(f.core.contiguous(), [u.contiguous() for u in f.factors], list(shape), f.ranks, f.order,
                      f.trunc, dtype, norm_sq, target, params)
