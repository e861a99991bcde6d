"""Seeded synthetic inputs shaped like the paper's workloads (host numpy, FP64).

This module is the ONLY code shared by the oracle side and the CUDA side. It
draws points and weights; it holds none of the method's arithmetic (no kernel,
no window, no FFT, no Sinkhorn step).

Seeding: numpy ``Generator(PCG64(SeedSequence([220107524, cfg_index, stream, seed])))``
with streams 0 = x, 1 = y, 2 = a, 3 = b, 4 = subsample indices, 5 = matvec
check rows, 6 = random test weights. Everything is generated
on the host, so the data is identical for any GPU count; a rank slices its
index range with :func:`shard_range`.

Distribution recipes (BASELINE.json configs; readings in DESIGN.md):
  uniform      U[0,1]^d
  normal_clip  N(0.5, s^2 I) clipped to [0,1]^d (s = 0.1 for d=1, 0.15 for d=3)
  gmm          k-component Gaussian mixture, equal component weights, means
               U[0,1]^d, isotropic sigma, clipped to [0,1]^d
  shell        uniform in the volume of the shell 0.3 <= |y - 1/2| <= 0.4
  jitter_grid  ((i + 1/2) + U(-0.4, 0.4)) / K per axis on a K x K grid
  pixel_grid   pixel centres (i + 1/2) / K of a K x K image (NEXT-1 image workloads)
Weights: uniform 1/n; dirichlet = Exp(1) normalised (Dirichlet(1));
bumps = smooth field of 32 Gaussian bumps at the pixel centre + 1e-6, normalised.
"""
from __future__ import annotations

import numpy as np

from .configs import Config, CONFIG_INDEX

SEED_ROOT = 220107524
STREAM_X, STREAM_Y, STREAM_A, STREAM_B, STREAM_SUB, STREAM_ROWS, STREAM_W = range(7)


def rng(cfg_index: int, stream: int, seed: int = 0) -> np.random.Generator:
    ss = np.random.SeedSequence([SEED_ROOT, int(cfg_index), int(stream), int(seed)])
    return np.random.Generator(np.random.PCG64(ss))


def _uniform(g, count, d):
    return g.random((count, d))


def _normal_clip(g, count, d, s):
    return np.clip(g.normal(0.5, s, size=(count, d)), 0.0, 1.0)


def _gmm(g, count, d, k, s):
    means = g.random((k, d))
    comp = g.integers(0, k, size=count)
    pts = g.normal(0.0, s, size=(count, d))
    pts += means[comp]
    np.clip(pts, 0.0, 1.0, out=pts)
    return pts


def _shell(g, count, r0=0.3, r1=0.4):
    v = g.normal(size=(count, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    r = (r0 ** 3 + g.random(count) * (r1 ** 3 - r0 ** 3)) ** (1.0 / 3.0)
    return 0.5 + v * r[:, None]


def _jitter_grid(g, K):
    i = np.arange(K, dtype=np.float64) + 0.5
    gx, gy = np.meshgrid(i, i, indexing="ij")
    pts = np.stack([gx.ravel(), gy.ravel()], axis=1)
    pts += g.uniform(-0.4, 0.4, size=pts.shape)
    pts /= K
    return pts


def _pixel_grid(K):
    """Pixel centres ((i + 1/2)/K, (j + 1/2)/K) of a K x K image, row-major (i slowest)."""
    i = (np.arange(K, dtype=np.float64) + 0.5) / K
    gx, gy = np.meshgrid(i, i, indexing="ij")
    return np.stack([gx.ravel(), gy.ravel()], axis=1)


def _bump_weights(g, pts_or_centres):
    """Smooth random field (32 Gaussian bumps) at the given points, + 1e-6, normalised."""
    nb = 32
    c = g.random((nb, 2))
    sb = g.uniform(0.03, 0.15, size=nb)
    amp = g.uniform(0.5, 1.5, size=nb)
    f = np.zeros(pts_or_centres.shape[0])
    for k in range(nb):
        r2 = ((pts_or_centres - c[k]) ** 2).sum(axis=1)
        f += amp[k] * np.exp(-r2 / (2.0 * sb[k] ** 2))
    f += 1e-6
    return f / f.sum()


def _points(cfg: Config, side: str, seed: int):
    ci = CONFIG_INDEX.get(cfg.name, 0)
    if side == "x":
        dist, count, stream, K = cfg.x_dist, cfg.n, STREAM_X, cfg.grid_x
    else:
        dist, count, stream, K = cfg.y_dist, cfg.m, STREAM_Y, cfg.grid_y
    g = rng(ci, stream, seed)
    d = cfg.d
    if dist == "uniform":
        return _uniform(g, count, d)
    if dist == "normal_clip":
        s = 0.1 if d == 1 else 0.15
        return _normal_clip(g, count, d, s)
    if dist == "gmm":
        return _gmm(g, count, d, cfg.gmm_k, cfg.gmm_sigma)
    if dist == "shell":
        assert d == 3
        return _shell(g, count)
    if dist == "jitter_grid":
        assert d == 2 and K * K == count
        return _jitter_grid(g, K)
    if dist == "pixel_grid":
        assert d == 2 and K * K == count
        return _pixel_grid(K)
    raise ValueError(dist)


def _weights(cfg: Config, side: str, count: int, seed: int):
    ci = CONFIG_INDEX.get(cfg.name, 0)
    stream = STREAM_A if side == "x" else STREAM_B
    g = rng(ci, stream, seed)
    if cfg.w_dist == "uniform":
        return np.full(count, 1.0 / count)
    if cfg.w_dist == "dirichlet":
        w = g.exponential(1.0, size=count)
        return w / w.sum()
    if cfg.w_dist == "bumps":
        K = cfg.grid_x if side == "x" else cfg.grid_y
        i = (np.arange(K, dtype=np.float64) + 0.5) / K
        gx, gy = np.meshgrid(i, i, indexing="ij")
        centres = np.stack([gx.ravel(), gy.ravel()], axis=1)
        return _bump_weights(g, centres)
    raise ValueError(cfg.w_dist)


def make_inputs(cfg: Config, seed: int = 0):
    """Return (x [n,d], y [m,d], a [n], b [m]) as C-contiguous float64 arrays."""
    x = np.ascontiguousarray(_points(cfg, "x", seed), dtype=np.float64)
    y = np.ascontiguousarray(_points(cfg, "y", seed), dtype=np.float64)
    a = np.ascontiguousarray(_weights(cfg, "x", x.shape[0], seed), dtype=np.float64)
    b = np.ascontiguousarray(_weights(cfg, "y", y.shape[0], seed), dtype=np.float64)
    return x, y, a, b


def subsample(cfg: Config, x, y, a, b, seed: int = 0):
    """Seeded subsample (sub_n, sub_m) with renormalised weights (divergence parity
    above 1e5 points, BASELINE.json north_star)."""
    ci = CONFIG_INDEX.get(cfg.name, 0)
    g = rng(ci, STREAM_SUB, seed)
    ix = np.sort(g.choice(x.shape[0], size=cfg.sub_n, replace=False))
    iy = np.sort(g.choice(y.shape[0], size=cfg.sub_m, replace=False))
    a2 = a[ix] / a[ix].sum()
    b2 = b[iy] / b[iy].sum()
    return (np.ascontiguousarray(x[ix]), np.ascontiguousarray(y[iy]),
            np.ascontiguousarray(a2), np.ascontiguousarray(b2))


def small_subsample(cfg: Config, x, y, a, b, k: int):
    """Seeded k-point subsample per side (stream 4, seed 1) with renormalised weights: the
    oracle-sized cases of the conditioning tests (dense oracle and fast-summation oracle run
    in seconds)."""
    ci = CONFIG_INDEX.get(cfg.name, 0)
    g = rng(ci, STREAM_SUB, 1)
    ix = np.sort(g.choice(x.shape[0], size=min(k, x.shape[0]), replace=False))
    iy = np.sort(g.choice(y.shape[0], size=min(k, y.shape[0]), replace=False))
    return (np.ascontiguousarray(x[ix]), np.ascontiguousarray(y[iy]),
            np.ascontiguousarray(a[ix] / a[ix].sum()), np.ascontiguousarray(b[iy] / b[iy].sum()))


def check_rows(cfg_index: int, count: int, total: int, seed: int = 0):
    """Seeded sorted target rows for sampled matvec parity (4096 above 1e5 points)."""
    g = rng(cfg_index, STREAM_ROWS, seed)
    if count >= total:
        return np.arange(total, dtype=np.int64)
    return np.sort(g.choice(total, size=count, replace=False)).astype(np.int64)


def uniform_test_weights(cfg_index: int, count: int, seed: int = 0):
    """Seeded U(0,1) weights for matvec checks."""
    return rng(cfg_index, STREAM_W, seed).random(count)


def shard_range(total: int, rank: int, world: int):
    """Contiguous balanced index range [lo, hi) of `rank` among `world` ranks."""
    base, rem = divmod(total, world)
    lo = rank * base + min(rank, rem)
    hi = lo + base + (1 if rank < rem else 0)
    return lo, hi
