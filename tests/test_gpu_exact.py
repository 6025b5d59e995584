"""GPU tests of the exact serial-sum engine (csrc/exact.cu): every sum the
encoder's decisions depend on must equal, bit for bit, the plain left-to-right
double loop of the reference (error_model.cpp:34-72, core_codec.cpp:131-155,
268-341, 405-411) -- checked against the one-thread serial chain on the device
and, for small cases, against a Python loop."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

INF = float("inf")


def hot_corner(n, seed, zeros=0.0):
    """magnitudes like a quantized Tucker core: max in [2^63, 2^64), decaying with index"""
    rng = np.random.default_rng(seed)
    x = np.abs(rng.standard_normal(n)) * np.exp(-np.linspace(0, 18, n)) * (1 + rng.random(n))
    x = x / x.max()
    m = np.floor(np.ldexp(x, 63) * 1.999).astype(np.uint64)
    if zeros:
        m[rng.random(n) < zeros] = 0
    return m


def tie_heavy(n, seed):
    """magnitudes with few significant bits: many exact ties in the sums"""
    rng = np.random.default_rng(seed)
    e = rng.integers(0, 62, n).astype(np.uint64)
    m = (np.uint64(1) << e) | ((np.uint64(1) << (e // np.uint64(2))) * rng.integers(0, 2, n).astype(np.uint64))
    return m.astype(np.uint64)


def py_serial(m, lo, hi, backward, term, plane, s0=0.0, need=INF, dec=None):
    """the reference's loops in Python doubles"""
    def sig2(v, p):
        if p == 0:
            return 0.0
        r = float(v & ((1 << p) - 1)) - float(1 << (p - 1))
        return r * r

    s = s0
    c0 = c1 = 0
    idx = range(hi - 1, lo - 1, -1) if backward else range(lo, hi)
    if need < INF and s >= need:
        return s, 0, 0, 1
    for i in idx:
        v = int(m[i])
        tb = v.bit_length() - 1
        if term == 0:
            c0 += tb <= plane
            c1 += tb == plane
            t = (float(v) * float(v) - sig2(v, plane)) if tb == plane else 0.0
        elif term == 1:
            c1 += tb > plane
            t = (sig2(v, plane + 1) - sig2(v, plane)) if tb > plane else 0.0
        elif term == 2:
            c0 += tb <= plane
            c1 += tb > plane
            t = (sig2(v, plane + 1) - sig2(v, plane)) if tb > plane else (
                (float(v) * float(v) - sig2(v, plane)) if tb == plane else 0.0)
        elif term == 3:
            t = float(v) * float(v)
        elif term == 4:
            if plane >= 64 or (v >> plane) == 0:
                r = float(v)
            elif plane == 0:
                r = 0.0
            else:
                r = float(v & ((1 << plane) - 1)) - float(1 << (plane - 1))
            t = r * r
        else:
            r = float(v) - float(int(dec[i]))
            t = r * r
        s = s + t
        if need < INF and s >= need:
            return s, c0, c1, 1
    return s, c0, c1, 0


def blocks(n, block):
    return [(b, min(n, b + block), 0, 0.0, INF) for b in range(0, n, block)]


def check_same(gpu_pkg, m, segs, kinds, dec=None):
    a = gpu_pkg.exact_sums(m, segs, kinds, dec=dec)
    b = gpu_pkg.exact_sums(m, segs, kinds, dec=dec, reference=True)
    for x, y in zip(a, b):
        assert np.array_equal(x, y), (x, y)
    return a


@pytest.mark.parametrize("n", [1, 5, 300, 4096, 20000])
def test_small_against_python_loop(gpu_pkg, n):
    m = hot_corner(n, n, zeros=0.1)
    segs = [(0, n, 0, 0.0, INF), (0, n, 1, 0.0, INF), (n // 3, n, 0, 12345.0, INF)]
    kinds = [(0, 60), (1, 60), (2, 55), (3, 0), (4, 50), (1, 3)]
    sums, c0, c1, cr = check_same(gpu_pkg, m, segs, kinds)
    for k, (t, p) in enumerate(kinds):
        for g, sg in enumerate(segs):
            ref = py_serial(m, sg[0], sg[1], sg[2], t, p, sg[3])
            assert sums[k, g] == ref[0] and c0[k, g] == ref[1] and c1[k, g] == ref[2], (k, g)


@pytest.mark.parametrize("gen,n,block", [("hot", 1 << 20, 16384), ("hot", 3_000_017, 65536), ("tie", 1 << 20, 1 << 18),
                                         ("hot0", 2_500_000, 40000)])
def test_block_stats_all_planes(gpu_pkg, gen, n, block):
    m = {"hot": lambda: hot_corner(n, 7), "tie": lambda: tie_heavy(n, 3),
         "hot0": lambda: hot_corner(n, 9, zeros=0.5)}[gen]()
    kinds = [(t, p) for p in range(63, 20, -3) for t in (0, 1)]
    check_same(gpu_pkg, m, blocks(n, block), kinds)


@pytest.mark.parametrize("n", [1 << 22, 9_000_001])
def test_whole_core_backward_sums(gpu_pkg, n):
    m = hot_corner(n, 11, zeros=0.2)
    rng = np.random.default_rng(1)
    dec = m & ~((np.uint64(1) << rng.integers(0, 40, n).astype(np.uint64)) - np.uint64(1))
    seg = [(0, n, 1, 0.0, INF)]
    for kind in [(3, 0), (4, 45), (4, 30), (5, 0)]:
        check_same(gpu_pkg, m, seg, [kind], dec=dec)


@pytest.mark.parametrize("term", [0, 1, 2])
def test_crossing_scans(gpu_pkg, term):
    n, block = 1 << 21, 1 << 19
    m = hot_corner(n, 5, zeros=0.1)
    p = 50
    tot = gpu_pkg.exact_sums(m, blocks(n, block), [(term, p)], reference=True)[0][0]
    segs = []
    for b, lo in enumerate(range(0, n, block)):
        for frac in (0.0, 1e-9, 0.3, 0.999999, 1.0, 1.5):
            cum = 1e30 * b
            segs.append((lo, min(n, lo + block), 0, cum, cum + frac * tot[b]))
    sums, c0, c1, cr = check_same(gpu_pkg, m, segs, [(term, p)])
    assert cr.sum() > 0 and (cr == 0).sum() > 0
    # python check on one crossing case
    sg = segs[2]
    ref = py_serial(m, sg[0], sg[1], 0, term, p, sg[3], sg[4])
    assert (sums[0, 2], c0[0, 2], c1[0, 2], cr[0, 2]) == ref


def test_signed_trail_sums_cross_zero(gpu_pkg):
    # trailing gains can be negative: sums that dip below zero and change sign
    n = 1 << 20
    rng = np.random.default_rng(2)
    p = 30
    hi = np.uint64(1) << np.uint64(p + 1)
    low = rng.integers(0, 1 << (p - 2), n).astype(np.uint64)  # low < 2^(p-2): negative gain when bit p set
    m = hi | (np.uint64(1) << np.uint64(p)) | low
    m[::7] = hi | low[::7]
    segs = [(0, n, 0, 0.0, INF), (0, n, 1, 0.0, INF), (0, n, 0, -1e20, INF), (0, n, 0, 2.0 ** 70, INF)]
    check_same(gpu_pkg, m, segs, [(1, p), (2, p)])


@pytest.mark.parametrize("gen,n,block,ptop,np_", [("hot", 3_000_017, 65536, 63, 32), ("hot0", 2_500_000, 40000, 50, 20),
                                                  ("tie", 1 << 20, 1 << 18, 40, 32)])
def test_plane_stats_lane_per_plane(gpu_pkg, gen, n, block, ptop, np_):
    """exact_plane_stats (one lane per plane, compact transducer) == the generic engine == the serial chain"""
    m = {"hot": lambda: hot_corner(n, 7), "tie": lambda: tie_heavy(n, 3),
         "hot0": lambda: hot_corner(n, 9, zeros=0.5)}[gen]()
    a = gpu_pkg.plane_stats(m, block, ptop, np_)
    kinds = [(t, ptop - l) for l in range(np_) for t in (0, 1)]
    b = gpu_pkg.exact_sums(m, blocks(n, block), kinds, reference=True)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
