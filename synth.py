"""Seeded synthetic inputs for the BASELINE.json configs (bench/test harness).

The paper's datasets are not available; these generators stand in for them
with the shapes, dtypes and value distributions BASELINE.json names.  All are
deterministic functions of (config, seed).  Coordinates are x = i / n.

  c1  64x64x64 fp32    8 separable sinusoid terms, amplitude N(0,1), + N(0,1e-3)
  c2  256^3 fp64       64 separable sinusoid terms, amplitude k^-1.5, + N(0,1e-5)
  c3  100x500x500 fp32 32 separable Gaussian blobs, + N(0,1e-3)
  c4  512x512x224 u16  blob abundance maps x 6-Gaussian spectra, clipped [0,1e4], rounded
  c5  1024^3 fp32      Gaussian random field, E(k) ~ k^-5/3 for k <= 341 (torch FFT on GPU)
"""
from __future__ import annotations

import numpy as np

CONFIGS = {
    "c1": dict(shape=(64, 64, 64), dtype="float32", res=(1e-3,)),
    "c2": dict(shape=(256, 256, 256), dtype="float64", res=(1e-2, 1e-4, 1e-6)),
    "c3": dict(shape=(100, 500, 500), dtype="float32", res=(1e-2, 1e-3, 1e-4)),
    "c4": dict(shape=(512, 512, 224), dtype="uint16", res=(1e-3,)),
    "c5": dict(shape=(1024, 1024, 1024), dtype="float32", res=(1e-2, 1e-3)),
}


def _separable(shape, amps, rng, out_dtype):
    """sum_k a_k v1_k (x) v2_k (x) v3_k as one GEMM: (V1 diag a) @ KhatriRao(V2, V3)^T."""
    K = len(amps)
    mats = [np.empty((n, K)) for n in shape]
    for k in range(K):
        for m, n in enumerate(shape):
            f = rng.uniform(0.5, 4.0)
            ph = rng.uniform(0.0, 2 * np.pi)
            x = np.arange(n, dtype=np.float64) / n
            mats[m][:, k] = np.sin(2 * np.pi * f * x + ph)
    rest = mats[1]
    for m in mats[2:]:
        rest = (rest[:, None, :] * m[None, :, :]).reshape(-1, K)
    return ((mats[0] * np.asarray(amps)[None, :]) @ rest.T).reshape(shape)


def sinusoids(shape, n_terms, decay=None, noise=1e-3, seed=0, dtype=np.float64):
    """Sum of separable sin(2 pi f x + phi) terms plus Gaussian noise (std `noise`)."""
    rng = np.random.default_rng(seed)
    if decay is None:
        amps = rng.standard_normal(n_terms)
    else:
        amps = np.arange(1, n_terms + 1, dtype=np.float64) ** (-decay)
    acc = _separable(shape, amps, rng, dtype)
    acc += noise * rng.standard_normal(shape)
    return acc.astype(dtype)


def blobs(shape, n_blobs=32, noise=1e-3, seed=0, dtype=np.float32):
    """Sum of axis-separable Gaussian blobs (centres U[0,1), widths U[0.02,0.2]), + noise."""
    rng = np.random.default_rng(seed)
    acc = np.zeros(shape, dtype=np.float64)
    for _ in range(n_blobs):
        a = rng.standard_normal()
        w = rng.uniform(0.02, 0.2)
        vecs = []
        for n in shape:
            c = rng.uniform(0.0, 1.0)
            x = np.arange(n, dtype=np.float64) / n
            vecs.append(np.exp(-0.5 * ((x - c) / w) ** 2))
        acc += a * np.einsum("i,j,k->ijk", *vecs)
    acc += noise * rng.standard_normal(shape)
    return acc.astype(dtype)


def spectral_cube(shape=(512, 512, 224), n_materials=8, seed=0):
    """Blob abundance maps x smooth 6-Gaussian spectra, scaled into [0, 1e4], uint16."""
    rng = np.random.default_rng(seed)
    nx, ny, nb = shape
    x = np.arange(nx) / nx
    y = np.arange(ny) / ny
    b = np.arange(nb, dtype=np.float64)
    acc = np.zeros(shape, dtype=np.float64)
    for _ in range(n_materials):
        amap = np.zeros((nx, ny))
        for _ in range(4):
            cx, cy = rng.uniform(0, 1, 2)
            w = rng.uniform(0.03, 0.25)
            amap += rng.uniform(0.2, 1.0) * np.outer(np.exp(-0.5 * ((x - cx) / w) ** 2),
                                                     np.exp(-0.5 * ((y - cy) / w) ** 2))
        spec = np.zeros(nb)
        for _ in range(6):
            mu = rng.uniform(0, nb)
            sd = rng.uniform(4, 40)
            spec += rng.uniform(0.1, 1.0) * np.exp(-0.5 * ((b - mu) / sd) ** 2)
        acc += np.einsum("ij,k->ijk", amap, spec)
    acc *= 1e4 / acc.max() * 1.05
    return np.rint(np.clip(acc, 0, 1e4)).astype(np.uint16)


def grf_torch(n=1024, kmax=341, seed=0, device="cuda"):
    """Gaussian random field with isotropic E(k) ~ k^-5/3 (k <= kmax), zero mean, unit variance."""
    import torch

    g = torch.Generator(device=device).manual_seed(seed)
    kx = torch.fft.fftfreq(n, d=1.0 / n, device=device)
    kz = torch.fft.rfftfreq(n, d=1.0 / n, device=device)
    out = torch.empty((n, n, n), dtype=torch.float32, device=device)
    spec = torch.empty((n, n, n // 2 + 1), dtype=torch.complex64, device=device)
    for i in range(n):  # slab-wise to bound memory
        k2 = kx[i] ** 2 + kx[:, None] ** 2 + kz[None, :] ** 2
        k = torch.sqrt(k2)
        amp = torch.where((k > 0) & (k <= kmax), k.clamp(min=1e-9) ** (-(5.0 / 3.0 + 2.0) / 2.0),
                          torch.zeros_like(k))
        re = torch.randn(k.shape, generator=g, device=device)
        im = torch.randn(k.shape, generator=g, device=device)
        spec[i] = torch.complex(re * amp, im * amp)
    out = torch.fft.irfftn(spec, s=(n, n, n))
    del spec
    out -= out.mean()
    out /= out.std()
    return out


def make(config: str, seed: int = 0):
    """Host numpy array for c1..c4 (c5 is generated on the GPU with grf_torch)."""
    if config == "c1":
        return sinusoids((64, 64, 64), 8, noise=1e-3, seed=seed, dtype=np.float32)
    if config == "c2":
        return sinusoids((256, 256, 256), 64, decay=1.5, noise=1e-5, seed=seed, dtype=np.float64)
    if config == "c3":
        return blobs((100, 500, 500), 32, noise=1e-3, seed=seed, dtype=np.float32)
    if config == "c4":
        return spectral_cube((512, 512, 224), seed=seed)
    raise ValueError(f"no host generator for {config}")


def small(kind: str, shape, seed=0, dtype=np.float64):
    """Reduced-size versions of the same families for parity tests."""
    if kind == "sin":
        return sinusoids(shape, 8, noise=1e-3, seed=seed, dtype=dtype)
    if kind == "sin_decay":
        return sinusoids(shape, 16, decay=1.5, noise=1e-5, seed=seed, dtype=dtype)
    if kind == "blobs":
        return blobs(shape, 12, noise=1e-3, seed=seed, dtype=dtype)
    if kind == "random":
        return np.random.default_rng(seed).uniform(-1, 1, shape).astype(dtype)
    raise ValueError(kind)
