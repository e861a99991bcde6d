"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle, element by element
on the same seeded inputs. Tolerances (BASELINE.json north_star): each fast-summation matvec
within relative l_inf 1e-9 of the direct sum; Sinkhorn divergence within relative 1e-8 where
the conditioning of Alg. 2 permits; stage kernels to FP64
roundoff of the window sums.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

from oracle import dense, nfft_ref
from synthetic import get, make_inputs, check_rows, uniform_test_weights
from synthetic.configs import CONFIG_INDEX

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def capi(cuda_ok):
    from paper_2201_07524_b200 import capi as C
    return C


@pytest.fixture(scope="module")
def ctx(capi):
    c = capi.Context(0)
    yield c
    c.close()


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def rel_linf(got, ref):
    return float(np.abs(got - ref).max() / np.abs(ref).max())


def sub(cfg, x, y, a, b, k, seed=0):
    """Deterministic first-k subsample with renormalised weights (oracle-sized cases)."""
    return x[:k], y[:k], a[:k] / a[:k].sum(), b[:k] / b[:k].sum()


# ------------------------------------------------------------------ stage kernels
@pytest.mark.parametrize("d,N,m_w,cnt", [(1, 64, 8, 257), (2, 32, 8, 131), (3, 16, 6, 67), (3, 16, 8, 33)])
def test_spread_interp_match_gridding_definition(capi, ctx, d, N, m_w, cnt):
    rng = np.random.default_rng(d * 100 + cnt)
    x, y = rng.random((cnt, d)), rng.random((cnt + 3, d))
    w = rng.random(cnt)
    P = capi.Plan(ctx, dev(x), dev(y), 20.0, N, 2.0, m_w)
    info = P.info()
    centre, rho, L = nfft_ref.geometry(x, y, 1 / 16)
    assert abs(info["rho"] - rho) <= 1e-15 * rho
    np.testing.assert_allclose(info["centre"][:d], centre, rtol=0, atol=1e-15)
    xs = nfft_ref.scale(x, centre, rho)
    n = int(info["n_grid"])
    g_ref = nfft_ref.grid_spread(xs, w, n, m_w, 2.0)
    g = capi.nfft_spread(P, 0, dev(w)).cpu().numpy()
    assert np.abs(g - g_ref).max() <= 1e-13 * np.abs(g_ref).max()
    G = rng.normal(size=(n,) * d)
    t_ref = nfft_ref.grid_interp(G, xs, m_w, 2.0)
    t = capi.nfft_interp(P, 0, dev(G)).cpu().numpy()
    scale = nfft_ref.grid_interp(np.abs(G), xs, m_w, 2.0)   # sum of |terms| per node
    assert (np.abs(t - t_ref) <= 1e-14 * scale).all()


@pytest.mark.parametrize("N,cnt,r", [(4096, 40, 2), (256, 200000, 2), (256, 50000, 1)])
def test_d1_spread_windows_match_gridding_definition(capi, ctx, N, cnt, r):
    """d = 1 spread (shared-memory window per CTA): sparse nodes on a large grid (windows wider
    than the shared buffer take the direct path), 2e5 nodes (full 256-node CTAs, ragged tail),
    and an r = 1 plan (position-sorted nodes) against the gridding definition. The grid
    geometry (rho, centre) is the plan's own, pinned by the test above."""
    rng = np.random.default_rng(N + cnt + r)
    x = np.sort(rng.random((cnt, 1)), axis=0)[::-1].copy() if r == 1 else rng.random((cnt, 1))
    y = rng.random((cnt + 5, 1))
    w = rng.random(cnt)
    kw = {"r": 1, "near_cells": 16} if r == 1 else {}
    P = capi.Plan(ctx, dev(x), dev(y), 20.0, N, 2.0, 8, **kw)
    info = P.info()
    xs = nfft_ref.scale(x, np.asarray(info["centre"][:1]), info["rho"])
    n = int(info["n_grid"])
    g_ref = nfft_ref.grid_spread(xs, w, n, 8, 2.0)
    g = capi.nfft_spread(P, 0, dev(w)).cpu().numpy()
    # u = n (x' + 1/2) carries |u| ulp ~ n 2^-53 of rounding on either side; the window's slope
    # turns it into ~1e-13 (n / 512) of phi(0) at n = 8192 (measured 3.6e-13)
    assert np.abs(g - g_ref).max() <= 1e-13 * max(1.0, n / 512) * np.abs(g_ref).max()


@pytest.mark.parametrize("case", ["single", "disjoint", "duplicates"])
def test_r1_d1_nearfield_edges(capi, ctx, case):
    """d = 1 near field edge cases against the oracle's statement of the method: one node per
    side, supports farther apart than the radius (no near pairs), and heavy duplication
    (runs of identical coordinates, equal fine keys)."""
    from oracle import laplace_ref as LR
    rng = np.random.default_rng(5)
    if case == "single":
        x, y = np.array([[0.3]]), np.array([[0.31]])
    elif case == "disjoint":
        x, y = 0.1 * rng.random((500, 1)), 0.9 + 0.1 * rng.random((400, 1))
    else:
        x = np.repeat(rng.random((40, 1)), 25, axis=0)
        y = np.repeat(rng.random((30, 1)), 33, axis=0)
    wy, wx = rng.random(y.shape[0]), rng.random(x.shape[0])
    P = capi.Plan(ctx, dev(x), dev(y), 20.0, 128, 2.0, 8, 1 / 16, 8, r=1, near_cells=16)
    for kernel in (0, 1):
        t = capi.fastsum_apply(P, dev(wy), 0, kernel).cpu().numpy()
        tt = capi.fastsum_apply(P, dev(wx), 1, kernel).cpu().numpy()
        ref = LR.fastsum_ndft(x, y, wy, 20.0, 128, 1 / 16, 8, 16, kernel=kernel)
        reft = LR.fastsum_ndft(y, x, wx, 20.0, 128, 1 / 16, 8, 16, kernel=kernel)
        # the window error is absolute, ~1e-15 ||w||_1 (the NFFT bound): on disjoint supports
        # the sums themselves are ~e^-16 ||w||_1, so the gate is on that scale, not on max |t|
        assert np.abs(t - ref).max() <= 1e-13 * np.abs(wy).sum(), (case, kernel, np.abs(t - ref).max())
        assert np.abs(tt - reft).max() <= 1e-13 * np.abs(wx).sum(), (case, kernel, np.abs(tt - reft).max())
        if case != "disjoint":
            assert rel_linf(t, ref) <= 1e-12 and rel_linf(tt, reft) <= 1e-12, (case, kernel, rel_linf(t, ref))


@pytest.mark.parametrize("d,m_w", [(3, 6), (2, 8)])
def test_cell_occupancies_match_gridding_definition(capi, ctx, d, m_w):
    """Clusters of x nodes confined to single grid cells, one cluster per occupancy in
    {1, 7, 8, 9, 16, 17, 24, 25, 31, 32, 33, 40, 64, 65, 97}: every per-cell batch shape of the
    tensor-core kernels (1..4 n-tiles of 8 nodes, full and ragged 32-node batches, several
    batches per cell) against the gridding definition. y holds the unit cube's corners, so the
    geometry is fixed and cell centres are known in advance."""
    rng = np.random.default_rng(7 + d)
    N = 16
    n = 2 * N
    L = 0.5 - 1 / 16
    rho = L / math.sqrt(d)
    occ = [1, 7, 8, 9, 16, 17, 24, 25, 31, 32, 33, 40, 64, 65, 97]
    lo, hi = int(math.ceil(n * (0.5 - rho / 2))) + 1, int(n * (0.5 + rho / 2)) - 2
    cells = set()
    while len(cells) < len(occ):
        cells.add(tuple(rng.integers(lo, hi, size=d)))
    pts = []
    for k, c in zip(occ, sorted(cells)):
        u = np.array(c, dtype=float) + 0.5 + rng.uniform(-0.35, 0.35, size=(k, d))   # inside the cell
        pts.append(0.5 + (u / n - 0.5) / rho)
    x = np.concatenate(pts)
    corners = np.array(np.meshgrid(*[[0.0, 1.0]] * d, indexing="ij")).reshape(d, -1).T
    y = np.concatenate([corners, rng.random((50, d))])
    P = capi.Plan(ctx, dev(x), dev(y), 20.0, N, 2.0, m_w)
    centre, rho_ref, _ = nfft_ref.geometry(x, y, 1 / 16)
    assert abs(P.info()["rho"] - rho_ref) <= 1e-15 * rho_ref and abs(rho_ref - rho) <= 1e-15 * rho
    xs = nfft_ref.scale(x, centre, rho_ref)
    cell_of = np.floor(n * (xs + 0.5)).astype(int)
    _, counts = np.unique(cell_of, axis=0, return_counts=True)
    assert sorted(counts.tolist()) == sorted(occ)
    G = rng.normal(size=(n,) * d)
    t_ref = nfft_ref.grid_interp(G, xs, m_w, 2.0)
    t = capi.nfft_interp(P, 0, dev(G)).cpu().numpy()
    scale = nfft_ref.grid_interp(np.abs(G), xs, m_w, 2.0)
    assert (np.abs(t - t_ref) <= 1e-14 * scale).all()
    w = rng.random(x.shape[0])
    g_ref = nfft_ref.grid_spread(xs, w, n, m_w, 2.0)
    g = capi.nfft_spread(P, 0, dev(w)).cpu().numpy()
    assert np.abs(g - g_ref).max() <= 1e-13 * np.abs(g_ref).max()
    P.close()


_VARIANT_SETS = {}


def _variant_sets():
    """Three d = 3 node sets on the unit cube's geometry (N = 16, n = 32): dense (3000 nodes in
    2^3 cells, ~375 per cell), mid (3000 in 3^3 cells, ~110 per cell) and sparse (300 spread
    over the box), with their oracle gridding results (computed once)."""
    if _VARIANT_SETS:
        return _VARIANT_SETS
    rng = np.random.default_rng(123)
    d, n, m_w = 3, 32, 6
    rho = (0.5 - 1 / 16) / math.sqrt(d)
    corners = np.array(np.meshgrid(*[[0.0, 1.0]] * d, indexing="ij")).reshape(d, -1).T
    y = np.concatenate([corners, rng.random((40, d))])
    for name, k, width in (("dense", 3000, 2), ("mid", 3000, 3), ("sparse", 300, 0)):
        if width:
            u = 15.0 + width * rng.random((k, d))   # cells 15 .. 15 + width - 1 per axis
            x = 0.5 + (u / n - 0.5) / rho
        else:
            x = 0.5 + (rng.random((k, d)) - 0.5) * 0.9
        centre, rho_ref, _ = nfft_ref.geometry(x, y, 1 / 16)
        xs = nfft_ref.scale(x, centre, rho_ref)
        w = rng.random(k)
        G = rng.normal(size=(n,) * d)
        _VARIANT_SETS[name] = (x, y, w, G, nfft_ref.grid_spread(xs, w, n, m_w, 2.0),
                               nfft_ref.grid_interp(G, xs, m_w, 2.0), nfft_ref.grid_interp(np.abs(G), xs, m_w, 2.0))
    return _VARIANT_SETS


@pytest.mark.parametrize("env", [{}, {"SK_SEG_DENSE_MIN": "0"}, {"SK_SEG_DENSE_MIN": "1000000000"},
                                 {"SK_XPAIRS": "1"}, {"SK_NO_DMMA": "1"}, {"SK_DETERMINISTIC": "1"},
                                 {"SK_DETERMINISTIC": "1", "SK_NO_DMMA": "1"}, {"SK_DETERMINISTIC": "0"},
                                 {"SK_SPREAD3_NOPIPE": "1"}])
def test_kernel_variants_match_gridding_definition(capi, ctx, env):
    """Every d = 3 spread/interp variant the plan can select (default shapes, forced dense or
    32-node segments, x-pair segments, the pair-barrier form of the pipelined spread, the vector path without tensor cores, the deterministic
    fixed-point accumulation on both) on dense, mid and sparse cells against the gridding
    definition."""
    sets = _variant_sets()
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        for name, (x, y, w, G, g_ref, t_ref, scale) in sets.items():
            P = capi.Plan(ctx, dev(x), dev(y), 20.0, 16, 2.0, 6)
            g = capi.nfft_spread(P, 0, dev(w)).cpu().numpy()
            assert np.abs(g - g_ref).max() <= 1e-13 * np.abs(g_ref).max(), (name, env)
            t = capi.nfft_interp(P, 0, dev(G)).cpu().numpy()
            assert (np.abs(t - t_ref) <= 1e-14 * scale).all(), (name, env)
            P.close()
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c5"])
def test_kernel_coefficients_match_oracle(capi, ctx, name):
    cfg = get(name)
    x, y, _, _ = make_inputs(cfg.with_(n=500, m=400) if cfg.n > 1000 else cfg)
    N = cfg.N if cfg.d < 3 else 32
    P = capi.Plan(ctx, dev(x), dev(y), cfg.lam, N, cfg.sigma, cfg.m_w, cfg.eps_B, cfg.p)
    info = P.info()
    for kernel in (0, 1):
        b = P.coefficients(kernel)
        ref = nfft_ref.bk_sampled(cfg.d, N, info["lambda_p"], info["rho"], kernel, info["L"], cfg.p).real
        assert np.abs(b - ref).max() <= 1e-14 * np.abs(ref).max()
        # accuracy report: the |b_k| of the (2N)^d sampling grid that the N-band drops (the +-N/2
        # faces count half, reading Q8), from the oracle's sampled K~ directly
        M = 2 * N
        g1 = (np.arange(M) - M // 2) / M
        xs = np.stack(np.meshgrid(*([g1] * cfg.d), indexing="ij"), axis=-1)
        Kt = nfft_ref.regularized_kernel(xs, info["lambda_p"], info["rho"], kernel, info["L"], cfg.p)
        B = np.abs(np.fft.fftn(np.fft.ifftshift(Kt))) / M ** cfg.d
        k1 = np.abs(np.fft.fftfreq(M, 1.0 / M))
        keep1 = np.where(k1 < N // 2, 1.0, np.where(k1 == N // 2, 0.5, 0.0))
        keep = keep1
        for _ in range(cfg.d - 1):
            keep = np.multiply.outer(keep, keep1)
        tail_ref = float((B * (1.0 - keep)).sum())
        # (entries near FFT rounding differ between the two FFTs: absolute slack at 1e-13 of sum |b|)
        assert abs(info["band_tail"][kernel] - tail_ref) <= 1e-6 * tail_ref + 1e-13 * B.sum(), \
            (kernel, info["band_tail"], tail_ref)


# ------------------------------------------------------------------ matvec parity
def _matvec_case(capi, ctx, cfg, x, y, a, b, rows_x, rows_y, weights, tol=1e-9):
    P = capi.Plan(ctx, dev(x), dev(y), cfg.lam, cfg.N, cfg.sigma, cfg.m_w, cfg.eps_B, cfg.p)
    worst = {}
    for kernel in (0, 1):
        for wname, (wy, wx) in weights.items():
            t = capi.fastsum_apply(P, dev(wy), 0, kernel).cpu().numpy()
            ref = dense.direct_sum(x, y, wy, cfg.lam, kernel, rows=rows_x)
            e1 = rel_linf(t[rows_x], ref)
            tt = capi.fastsum_apply(P, dev(wx), 1, kernel).cpu().numpy()
            reft = dense.direct_sum(y, x, wx, cfg.lam, kernel, rows=rows_y)
            e2 = rel_linf(tt[rows_y], reft)
            worst[(kernel, wname)] = (e1, e2)
    return worst


@pytest.mark.parametrize("name,n_rows", [("c1", None), ("c2", None)])
def test_matvec_parity_full_size(capi, ctx, name, n_rows):
    """Full-size plans; full matvecs against the direct sum for the configs with n, m <= 1e5
    (c1, c2: BJ's protocol compares every row there). c3-c5 run BJ's 4096-row protocol against
    oracle goldens in test_gpu_protocol.py."""
    cfg = get(name)
    x, y, a, b = make_inputs(cfg)
    ci = CONFIG_INDEX[name]
    rx = check_rows(ci, n_rows or x.shape[0], x.shape[0])
    ry = check_rows(ci, n_rows or y.shape[0], y.shape[0], seed=1)
    weights = {"marginal": (b, a), "uniform01": (uniform_test_weights(ci, y.shape[0]), uniform_test_weights(ci, x.shape[0], 1))}
    worst = _matvec_case(capi, ctx, cfg, x, y, a, b, rx, ry, weights)
    bad = {k: v for k, v in worst.items() if max(v) > 1e-9}
    # c1 at N = 64: the c*exp(-lam c) kernel is truncated at exp(-pi^2 32^2/lam') ~ 1e-9
    # (the plan's band tail reports it); the Gaussian kernel passes.
    if name == "c1":
        bad = {k: v for k, v in bad.items() if k[0] == 0}
    assert not bad, worst


def test_matvec_parity_c1_converged_weights(capi, ctx):
    """Weights (iii): the oracle's converged scalings v = exp(lam g), u = exp(lam f).
    At BJ's N = 64 the K v direction meets 1e-9 but K^T u does not: u spans e^{lam range(f)}
    and the Fourier truncation error exp(-pi^2 32^2/lam') ~ 1e-9 * ||u||_1 exceeds 1e-9 max t~
    (DESIGN.md "Conditioning"). At N = 96 (the documented c1 deviation) every case passes."""
    cfg = get("c1")
    x, y, a, b = make_inputs(cfg)
    f, g = dense.sinkhorn_log(x, y, a, b, cfg.lam, cfg.iters)
    v, u = np.exp(cfg.lam * g), np.exp(cfg.lam * f)
    rx, ry = np.arange(x.shape[0]), np.arange(y.shape[0])
    worst = _matvec_case(capi, ctx, cfg, x, y, a, b, rx, ry, {"converged": (v, u)})
    assert worst[(0, "converged")][0] <= 1e-9, worst
    assert max(worst[(0, "converged")]) <= 1e-8, worst
    worst96 = _matvec_case(capi, ctx, cfg.with_(N=96), x, y, a, b, rx, ry, {"converged": (v, u)})
    assert max(max(e) for e in worst96.values()) <= 1e-9, worst96


# ------------------------------------------------------------------ Sinkhorn divergence parity
def _gpu_divergence(capi, ctx, cfg, x, y, a, b, N=None, iters=None):
    P = capi.Plan(ctx, dev(x), dev(y), cfg.lam, N or cfg.N, cfg.sigma, cfg.m_w, cfg.eps_B, cfg.p)
    da, db = dev(a), dev(b)
    u, v, info = capi.sinkhorn_run(P, da, db, iters or cfg.iters)
    sd, sc = capi.sinkhorn_divergence(P, da, db, u, v)
    return sd, sc, info, P, u, v


def test_divergence_parity_c1_N96(capi, ctx):
    """c1 workload at N = 96 (documented deviation from BJ's N = 64): s~ and s
    within 1e-8 relative of the dense log-domain oracle."""
    cfg = get("c1")
    x, y, a, b = make_inputs(cfg)
    ref, _, _ = dense.sinkhorn_divergence(x, y, a, b, cfg.lam, cfg.iters)
    sd, sc, info, *_ = _gpu_divergence(capi, ctx, cfg, x, y, a, b, N=96)
    assert abs(sc - ref["s_cost"]) <= 1e-8 * abs(ref["s_cost"]), (sc, ref, info.asdict())
    assert abs(sd - ref["s_dual"]) <= 1e-8 * abs(ref["s_dual"]), (sd, ref, info.asdict())


@pytest.mark.parametrize("name,k", [("c2", 3000), ("c3", 3000), ("c5", 3000)])
def test_divergence_parity_subsample(capi, ctx, name, k):
    """Oracle-sized subsamples (first k points, renormalised weights) of each workload at the
    config's lam and NFFT parameters."""
    cfg = get(name)
    gen_cfg = cfg.with_(n=min(cfg.n, 20000), m=min(cfg.m, 20000))
    x, y, a, b = sub(cfg, *make_inputs(gen_cfg), k)
    ref, _, _ = dense.sinkhorn_divergence(x, y, a, b, cfg.lam, cfg.iters)
    sd, sc, info, *_ = _gpu_divergence(capi, ctx, cfg, x, y, a, b)
    err = abs(sc - ref["s_cost"]) / abs(ref["s_cost"])
    # c2 (lam = 50, Dirichlet weights) is conditioning-limited (kappa up to 1e14): gate on the
    # method's envelope there, 1e-8 elsewhere.
    tol = 1e-8 if name != "c2" else 1e-5
    assert err <= tol, (name, sc, ref, info.asdict())


def test_adjointness_and_gauge(capi, ctx):
    cfg = get("c3").with_(n=5000, m=4000)
    x, y, a, b = make_inputs(cfg)
    P = capi.Plan(ctx, dev(x), dev(y), cfg.lam, cfg.N, cfg.sigma, cfg.m_w, cfg.eps_B, cfg.p)
    rng = np.random.default_rng(0)
    uu, vv = dev(rng.random(x.shape[0])), dev(rng.random(y.shape[0]))
    lhs = float(uu @ capi.fastsum_apply(P, vv, 0, 0))
    rhs = float(capi.fastsum_apply(P, uu, 1, 0) @ vv)
    assert abs(lhs - rhs) <= 1e-13 * abs(lhs)
    da, db = dev(a), dev(b)
    u, v, _ = capi.sinkhorn_run(P, da, db, 30)
    s1 = capi.sinkhorn_divergence(P, da, db, u, v)
    s2 = capi.sinkhorn_divergence(P, da, db, u * 1e3, v / 1e3)
    assert abs(s1[0] - s2[0]) <= 1e-12 * abs(s1[0]) and abs(s1[1] - s2[1]) <= 1e-12 * abs(s1[1])
    # rescale policies are pure gauge (Eq. (scale), reading Q4)
    u3, v3, _ = capi.sinkhorn_run(P, da, db, 30, rescale_policy=1)
    s3 = capi.sinkhorn_divergence(P, da, db, u3, v3)
    assert abs(s1[1] - s3[1]) <= 1e-11 * abs(s1[1])


def test_single_source_closed_form(capi, ctx):
    """n = 1 (pin P2): s~ = sum_j b_j |x1 - y_j|^2, s = s~ - H(b)/lam."""
    rng = np.random.default_rng(3)
    x, y = rng.random((1, 2)), rng.random((777, 2))
    b = rng.random(777)
    b /= b.sum()
    lam = 10.0
    P = capi.Plan(ctx, dev(x), dev(y), lam, 128, 2.0, 8)
    u, v, _ = capi.sinkhorn_run(P, dev(np.ones(1)), dev(b), 3)
    sd, sc = capi.sinkhorn_divergence(P, dev(np.ones(1)), dev(b), u, v)
    s_cost = float((b * ((x - y) ** 2).sum(1)).sum())
    H = -float((b * np.log(b)).sum())
    assert abs(sc - s_cost) <= 1e-10 * s_cost
    assert abs(sd - (s_cost - H / lam)) <= 1e-10 * abs(s_cost - H / lam)


def test_errors(capi, ctx):
    x = np.random.default_rng(0).random((10, 2))
    xb = x.copy()
    xb[3, 1] = np.nan
    with pytest.raises(capi.SkError) as e:
        capi.Plan(ctx, dev(xb), dev(x), 10.0, 32)
    assert e.value.code == capi.SK_EGEOMETRY
    with pytest.raises(capi.SkError) as e:
        capi.Plan(ctx, dev(x), dev(x), -1.0, 32)
    assert e.value.code == capi.SK_EINVAL
    with pytest.raises(capi.SkError) as e:
        capi.Plan(ctx, dev(x), dev(x), 1.0, 33)
    assert e.value.code == capi.SK_EINVAL
    with pytest.raises(capi.SkError) as e:
        capi.Plan(ctx, dev(x), dev(x), 1.0, 8, 2.0, 8)   # sigma N = 16 < 4 m_w
    assert e.value.code == capi.SK_EINVAL
    x3 = np.random.default_rng(1).random((10, 3))
    with pytest.raises(capi.SkError) as e:
        capi.Plan(ctx, dev(x3), dev(x3), 1.0, 1292, 2.0, 6)   # (sigma N)^3 = 2584^3 > 2^31 cells
    assert e.value.code == capi.SK_EINVAL


def test_weights_are_validated(capi, ctx):
    """sinkhorn_run rejects weights that are not > 0 or do not sum to 1 +- 1e-12
    (SK_EINVAL), on either side; valid weights run and report both conditioning estimates."""
    cfg = get("c3").with_(n=3000, m=2500)
    x, y, a, b = make_inputs(cfg)
    a, b = a / a.sum(), b / b.sum()
    P = capi.Plan(ctx, dev(x), dev(y), cfg.lam, cfg.N, cfg.sigma, cfg.m_w, cfg.eps_B, cfg.p)
    a0 = a.copy()
    a0[5] = 0.0
    a0 /= a0.sum()
    bneg = b.copy()
    bneg[7] = -bneg[7]
    bneg /= bneg.sum()
    for aa, bb in ((a * 1.001, b), (a, b * (1 - 1e-9)), (a0, b), (a, bneg), (a * np.nan, b)):
        with pytest.raises(capi.SkError) as e:
            capi.sinkhorn_run(P, dev(aa), dev(bb), 3)
        assert e.value.code == capi.SK_EINVAL, str(e.value)
    u, v, info = capi.sinkhorn_run(P, dev(a), dev(b), 3)
    assert info.bad_iter == -1 and info.bad_side == -1
    assert np.isfinite(info.kappa_log10_est) and np.isfinite(info.kappa_u_log10_est)


@pytest.mark.parametrize("iters", [1, 6])
@pytest.mark.parametrize("case", ["both_sides", "v_side"])
def test_enonpos_single_event(capi, ctx, iters, case):
    """SK_ENONPOS (tau_pos = 1e-300): nodes farther than sqrt(700 / lam) from every
    atom of the other measure have K v (or K^T u) below 1e-300, so the fast summation returns
    rounding-level values of either sign there. iters = 1 runs eagerly, iters = 6 replays
    iterations 0..4 as a CUDA graph (the iteration number then comes from the device counter).
    The report is one event: the earliest iteration, u-update before v-update.
      both_sides: x in [0, 0.1], y in [1.0, 1.1], lam = 2000: the first u-update fails (side 0,
        iteration 0) at an x node;
      v_side: the x nodes sit inside the y cluster, plus 40 y nodes at 1.5: every K v is fine,
        the first v-update fails (side 1, iteration 0) at one of the far y nodes."""
    rng = np.random.default_rng(11)
    lam = 2000.0
    if case == "both_sides":
        x = rng.uniform(0.0, 0.1, size=(60, 1))
        y = rng.uniform(1.0, 1.1, size=(50, 1))
        far_side, far = 0, np.arange(60)
    else:
        x = rng.uniform(0.0, 0.1, size=(60, 1))
        y = np.concatenate([rng.uniform(0.0, 0.1, size=(50, 1)), rng.uniform(1.5, 1.52, size=(40, 1))])
        far_side, far = 1, np.arange(50, 90)
    a, b = np.full(x.shape[0], 1.0 / x.shape[0]), np.full(y.shape[0], 1.0 / y.shape[0])
    P = capi.Plan(ctx, dev(x), dev(y), lam, 256, 2.0, 8)
    with pytest.raises(capi.SkError) as e:
        capi.sinkhorn_run(P, dev(a), dev(b), iters)
    assert e.value.code == capi.SK_ENONPOS, str(e.value)
    info = e.value.info
    assert info.bad_iter == 0 and info.bad_side == far_side and info.bad_rank == 0, info.asdict()
    assert info.bad_index in far, info.asdict()


def test_host_buffer_solve_matches_device(capi, ctx):
    cfg = get("c3").with_(n=20000, m=15000)
    x, y, a, b = make_inputs(cfg)
    a, b = a / a.sum(), b / b.sum()
    h = capi.sinkhorn_solve(ctx, x, y, a, b, cfg.lam, cfg.N, cfg.sigma, cfg.m_w, iters=30, inputs_on_host=True)
    d_ = capi.sinkhorn_solve(ctx, dev(x), dev(y), dev(a), dev(b), cfg.lam, cfg.N, cfg.sigma, cfg.m_w, iters=30)
    # identical inputs; only the order of the FP64 atomics in the spread flush differs
    # (well-conditioned workload, kappa ~ 10^1.6, so rounding is not amplified)
    assert abs(h[0] - d_[0]) <= 1e-12 * abs(h[0]) and abs(h[1] - d_[1]) <= 1e-12 * abs(h[1])


@pytest.mark.parametrize("name,n,m", [("c1", 1000, 1000), ("c2", 20000, 15000), ("c5", 200000, 160000)])
def test_box_exchange_is_exact(capi, ctx, name, n, m):
    """a3 exchange over the touched box only: with SK_FORCE_BOX_EXCHANGE a
    one-rank plan packs the box, clears the whole grid and unpacks it before the FFT, so the
    matvec is bit-identical iff the box holds every nonzero of the spread grid."""
    cfg = get(name)
    x, y, a, b = make_inputs(cfg.with_(n=n, m=m) if cfg.n > n else cfg)
    P0 = capi.Plan(ctx, dev(x), dev(y), cfg.lam, cfg.N, cfg.sigma, cfg.m_w, cfg.eps_B, cfg.p)
    os.environ["SK_FORCE_BOX_EXCHANGE"] = "1"
    try:
        P1 = capi.Plan(ctx, dev(x), dev(y), cfg.lam, cfg.N, cfg.sigma, cfg.m_w, cfg.eps_B, cfg.p)
    finally:
        del os.environ["SK_FORCE_BOX_EXCHANGE"]
    info = P1.info()
    n_grid = int(info["n_grid"])
    assert info["box_size"] == int(np.prod(info["box_n"][:cfg.d]))
    assert info["box_size"] < n_grid ** cfg.d
    # the spread grid is zero outside the box
    g = capi.nfft_spread(P1, 1, dev(b)).cpu().numpy()
    sl = tuple(slice(lo, lo + k) for lo, k in zip(info["box_lo"][:cfg.d], info["box_n"][:cfg.d]))
    inside = np.zeros(g.shape, bool)
    inside[sl] = True
    assert np.all(g[~inside] == 0.0) and np.any(g[inside] != 0.0)
    for tr, w in ((0, b), (1, a)):
        for kernel in (0, 1):
            t0 = capi.fastsum_apply(P0, dev(w), tr, kernel).cpu().numpy()
            t1 = capi.fastsum_apply(P1, dev(w), tr, kernel).cpu().numpy()
            # same data; only the order of the spread's FP64 atomics may differ
            assert np.abs(t0 - t1).max() <= 1e-13 * np.abs(t0).max()


# ------------------------------------------------------------------ NEXT-1: image workloads (lambda = 20)
@pytest.mark.parametrize("name", ["img32", "img64"])
def test_image_divergence_parity(capi, ctx, name):
    """two K x K bump-field images on the pixel grid at the paper's
    lambda = 20 (Tables 3, 6, 7). Well conditioned, so the GPU's s~ and s match
    the dense oracle far inside the BJ gate (the paper reports agreement to 13-14 digits,
    P:L1088-1091)."""
    cfg = get(name)
    x, y, a, b = make_inputs(cfg)
    ref, _, _ = dense.sinkhorn_divergence(x, y, a, b, cfg.lam, cfg.iters)
    sd, sc, info, *_ = _gpu_divergence(capi, ctx, cfg, x, y, a, b)
    assert abs(sc - ref["s_cost"]) <= 1e-10 * abs(ref["s_cost"]), (sc, ref, info.asdict())
    assert abs(sd - ref["s_dual"]) <= 1e-10 * abs(ref["s_dual"]), (sd, ref, info.asdict())


@pytest.mark.parametrize("name", ["img128", "img512"])
def test_image_matvec_parity(capi, ctx, name):
    cfg = get(name)
    x, y, a, b = make_inputs(cfg)
    ci = CONFIG_INDEX[name]
    rx = check_rows(ci, 4096, x.shape[0])
    ry = check_rows(ci, 4096, y.shape[0], seed=1)
    weights = {"marginal": (b, a), "uniform01": (uniform_test_weights(ci, y.shape[0]), uniform_test_weights(ci, x.shape[0], 1))}
    worst = _matvec_case(capi, ctx, cfg, x, y, a, b, rx, ry, weights)
    assert max(max(v) for v in worst.values()) <= 1e-9, worst


# ------------------------------------------------------------------ NEXT-3: diagnostics, stopping, lambda sweep
def _c1_small():
    cfg = get("c1")
    x, y, a, b = make_inputs(cfg)
    return cfg, x[:400], y[:300], a[:400] / a[:400].sum(), b[:300] / b[:300].sum()


def test_trace_matches_oracle(capi, ctx):
    """Per-iteration residuals ||E||_1 (Eq. (Error)), KL terms (Lemma P:L353) and
    sum p log alpha of the GPU run against oracle.diagnostics on the same inputs."""
    from oracle import diagnostics as D
    cfg, x, y, a, b = _c1_small()
    lam, iters = 30.0, 25
    ref, al, at = D.sinkhorn_trace(x, y, a, b, lam, iters)
    P = capi.Plan(ctx, dev(x), dev(y), lam, cfg.N, cfg.sigma, cfg.m_w, cfg.eps_B, cfg.p)
    u, v, info, tr = capi.sinkhorn_run_trace(P, dev(a), dev(b), iters)
    assert info.iters_done == iters and tr.shape == ref.shape
    err = np.abs(tr - ref)
    assert (err <= 1e-9 * np.maximum(1.0, np.abs(ref)) + 1e-12).all(), (err.max(axis=0), ref[-1], tr[-1])
    # the run itself is unchanged by tracing (up to the order of the spread's FP64 atomics)
    u2, v2, _ = capi.sinkhorn_run(P, dev(a), dev(b), iters)
    assert float(((u - u2).abs() / u2).max()) < 1e-11 and float(((v - v2).abs() / v2).max()) < 1e-11


def test_residual_stopping_matches_oracle(capi, ctx):
    """tol > 0 (reading Q5): stop after the first iteration whose residual ||pi 1 - p||_1 (measured
    at its u-update) is <= tol; the oracle's trace fixes which iteration that is."""
    from oracle import diagnostics as D
    cfg, x, y, a, b = _c1_small()
    lam, tol = 30.0, 1e-7
    ref, *_ = D.sinkhorn_trace(x, y, a, b, lam, 60)
    want = next(it + 1 for it in range(60) if ref[it, 0] <= tol)
    P = capi.Plan(ctx, dev(x), dev(y), lam, cfg.N, cfg.sigma, cfg.m_w, cfg.eps_B, cfg.p)
    u, v, info = capi.sinkhorn_run(P, dev(a), dev(b), 60, tol=tol)
    assert info.iters_done == want and info.residual <= tol
    with pytest.raises(capi.SkError) as e:
        capi.sinkhorn_run(P, dev(a), dev(b), 3, tol=1e-14)
    assert e.value.code == capi.SK_ENOTCONVERGED


@pytest.mark.parametrize("lam", [5.0, 10.0, 15.0, 20.0, 25.0])
def test_lambda_sweep_sandwich(capi, ctx, lam):
    """Fig. 3: n = n~ = 1000 at lambda in {5, ..., 25}, r = 2 (d = 1, c1 inputs).
    GPU s and s~ equal the oracle's, and s <= W_2^2 <= s~ with W_2^2 from the exact 1-D
    quantile formula (Prop. 3.3 sandwich). N = 128: at lambda = 5 the kernel is still
    e^-5 at the regularisation radius L, and N = 64 leaves a 2e-8 fast-summation error
    (oracle.nfft_ref.fastsum_ndft, the method's own error); N = 128 gives 4e-11."""
    from oracle import exact_ot
    cfg = get("c1")
    x, y, a, b = make_inputs(cfg)
    ref, _, _ = dense.sinkhorn_divergence(x, y, a, b, lam, 300)
    sd, sc, info, *_ = _gpu_divergence(capi, ctx, cfg.with_(lam=lam, N=128), x, y, a, b, iters=300)
    assert abs(sc - ref["s_cost"]) <= 1e-9 * abs(ref["s_cost"]), (lam, sc, ref)
    assert abs(sd - ref["s_dual"]) <= 1e-9 * abs(ref["s_dual"]), (lam, sd, ref)
    W = exact_ot.w2_1d(x[:, 0], a, y[:, 0], b)
    assert sd <= W <= sc


# ------------------------------------------------------------------ multi-rank code paths on one GPU
def test_emulated_two_rank_world(capi):
    """SK_EMULATE_WORLD=2: two ranks with identical shards (x, y, weights a/2, b/2 on each), i.e.
    every atom duplicated with half its mass. Every multi-rank path runs (global counts via the
    sum all-reduce, box exchange of the grid, scalar all-reduces). Exact consequences:
    K_global v = 2 K v; the Sinkhorn iterates are U = u/4, V = v at every iteration, so
    s~ is unchanged and s drops by log(4)/lambda (Eq. (14) P:L211 with sum p = 1)."""
    cfg = get("c3").with_(n=20000, m=15000)
    x, y, a, b = make_inputs(cfg)
    a, b = a / a.sum(), b / b.sum()
    iters = 20
    c1 = capi.Context(0)
    P1 = capi.Plan(c1, dev(x), dev(y), cfg.lam, cfg.N, cfg.sigma, cfg.m_w, cfg.eps_B, cfg.p)
    w = dev(uniform_test_weights(3, y.shape[0]))
    t1 = capi.fastsum_apply(P1, w, 0, 0)
    u1, v1, _ = capi.sinkhorn_run(P1, dev(a), dev(b), iters)
    sd1, sc1 = capi.sinkhorn_divergence(P1, dev(a), dev(b), u1, v1)
    os.environ["SK_EMULATE_WORLD"] = "2"
    try:
        c2 = capi.Context(0)
    finally:
        del os.environ["SK_EMULATE_WORLD"]
    P2 = capi.Plan(c2, dev(x), dev(y), cfg.lam, cfg.N, cfg.sigma, cfg.m_w, cfg.eps_B, cfg.p)
    info = P2.info()
    assert info["total_x"] == 2 * x.shape[0] and info["total_y"] == 2 * y.shape[0]
    t2 = capi.fastsum_apply(P2, w, 0, 0)
    assert float(((t2 - 2 * t1).abs()).max() / t1.abs().max()) < 1e-13
    u2, v2, _ = capi.sinkhorn_run(P2, dev(a / 2), dev(b / 2), iters)
    assert float(((4 * u2 - u1).abs() / u1).max()) < 1e-11 and float(((v2 - v1).abs() / v1).max()) < 1e-11
    sd2, sc2 = capi.sinkhorn_divergence(P2, dev(a / 2), dev(b / 2), u2, v2)
    assert abs(sc2 - sc1) <= 1e-11 * abs(sc1)
    assert abs(sd2 - (sd1 - math.log(4) / cfg.lam)) <= 1e-11 * abs(sd1)
    for P, c in ((P1, c1), (P2, c2)):
        P.close()
        c.close()


@pytest.mark.parametrize("d,N", [(1, 128), (2, 64), (3, 32)])
def test_r1_across_ranks(capi, d, N):
    """r = 1 across ranks (include/sinkhorn_nfft.h): the near field gathers every rank's sources.
    SK_EMULATE_WORLD=2 (two identical shards, every atom duplicated): K_global v = 2 K v for both
    kernels and directions, exactly as the far field's grid all-reduce; a one-rank NCCL
    communicator runs the coordinate and weight all-gathers (ncclBroadcast) as the identity and
    equals the communicator-free plan. d = 1 takes the position-sorted near-field kernel, d = 2, 3
    the tiled one."""
    rng = np.random.default_rng(40 + d)
    n, m = 3000, 2500
    x = 0.5 + 0.2 * rng.normal(size=(n, d))
    y = rng.random((m, d))
    wy, wx = rng.random(m), rng.random(n)
    kw = dict(r=1, near_cells=16 if d < 3 else 6)

    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)

    def applies(c, scale=1.0):
        P = capi.Plan(c, dev(x), dev(y), 20.0, N, 2.0, 8 if d < 3 else 6, **kw)
        out = [capi.fastsum_apply(P, dev(w), tr, k).cpu().numpy() for k in (0, 1) for tr, w in ((0, wy), (1, wx))]
        u, v, _ = capi.sinkhorn_run(P, dev(a * scale), dev(b * scale), 8)   # graph-captured gathers
        out += [u.cpu().numpy(), v.cpu().numpy()]
        P.close()
        return out
    c1 = capi.Context(0)
    ref = applies(c1)
    os.environ["SK_EMULATE_WORLD"] = "2"
    try:
        c2 = capi.Context(0)
    finally:
        del os.environ["SK_EMULATE_WORLD"]
    emu = applies(c2, 0.5)   # every atom duplicated with half its mass: U = u / 4, V = v
    for i, (t2, t1) in enumerate(zip(emu[:4], ref[:4])):
        assert rel_linf(t2, 2 * t1) <= 1e-13, (d, i, rel_linf(t2, 2 * t1))
    assert rel_linf(4 * emu[4], ref[4]) <= 1e-11 and rel_linf(emu[5], ref[5]) <= 1e-11
    c3 = capi.Context(0, 0, 1, capi.sk_nccl_unique_id())
    for i, (t3, t1) in enumerate(zip(applies(c3), ref)):
        assert rel_linf(t3, t1) <= (1e-13 if i < 4 else 1e-11), (d, i, rel_linf(t3, t1))
    for c in (c3, c2, c1):
        c.close()


def test_nccl_one_rank_path(capi):
    """world_size 1 with an ncclUniqueId: a real one-rank NCCL communicator, so the bbox min/max,
    the box exchange of every fast summation and the scalar sums all run through ncclAllReduce
    (dlopen'ed libnccl, inside the CUDA-graph capture of sinkhorn_run) as the identity. Results
    equal the communicator-free context's to summation-order rounding."""
    cfg = get("c3").with_(n=20000, m=15000)
    x, y, a, b = make_inputs(cfg)
    iters = 20
    c1 = capi.Context(0)
    c2 = capi.Context(0, 0, 1, capi.sk_nccl_unique_id())
    out = []
    for c in (c1, c2):
        P = capi.Plan(c, dev(x), dev(y), cfg.lam, cfg.N, cfg.sigma, cfg.m_w, cfg.eps_B, cfg.p)
        w = dev(uniform_test_weights(3, y.shape[0]))
        t = capi.fastsum_apply(P, w, 0, 0)
        u, v, _ = capi.sinkhorn_run(P, dev(a), dev(b), iters)
        sd, sc = capi.sinkhorn_divergence(P, dev(a), dev(b), u, v)
        out.append((t, u, v, sd, sc, P.info()))
        P.close()
    (t1, u1, v1, sd1, sc1, i1), (t2, u2, v2, sd2, sc2, i2) = out
    assert i2["box_size"] == i1["box_size"] and i2["total_x"] == x.shape[0]
    assert float(((t2 - t1).abs()).max() / t1.abs().max()) < 1e-13
    assert float(((u2 - u1).abs() / u1).max()) < 1e-11 and float(((v2 - v1).abs() / v1).max()) < 1e-11
    assert abs(sd2 - sd1) <= 1e-11 * abs(sd1) and abs(sc2 - sc1) <= 1e-11 * abs(sc1)
    c2.close()
    c1.close()


# ------------------------------------------------------------------ NEXT-2: r = 1 (Laplace kernel + near field)
@pytest.mark.parametrize("d,n,N", [(1, 300, 128), (2, 150, 128)])
def test_r1_fastsum_matches_oracle(capi, ctx, d, n, N):
    """fastsum_plan_ex with r = 1: the GPU fast summation equals the oracle's statement of the
    same method (laplace_ref.fastsum_ndft: exact NDFTs of K_R's b_k plus the brute-force near
    field) to the window error, and the direct sum to the method error (both kernels, both
    directions)."""
    from oracle import laplace_ref as LR
    rng = np.random.default_rng(10 + d)
    x, y = rng.random((n, d)), rng.random((n + 7, d))
    wy, wx = rng.random(n + 7), rng.random(n)
    lam = 20.0
    P = capi.Plan(ctx, dev(x), dev(y), lam, N, 2.0, 8, 1 / 16, 8, r=1, near_cells=16)
    for kernel in (0, 1):
        t = capi.fastsum_apply(P, dev(wy), 0, kernel).cpu().numpy()
        tt = capi.fastsum_apply(P, dev(wx), 1, kernel).cpu().numpy()
        m_ref = LR.fastsum_ndft(x, y, wy, lam, N, 1 / 16, 8, 16, kernel=kernel)
        mt_ref = LR.fastsum_ndft(y, x, wx, lam, N, 1 / 16, 8, 16, kernel=kernel)
        assert rel_linf(t, m_ref) <= 1e-12 and rel_linf(tt, mt_ref) <= 1e-12, (kernel, rel_linf(t, m_ref))
        ref = dense.direct_sum(x, y, wy, lam, kernel, r=1)
        reft = dense.direct_sum(y, x, wx, lam, kernel, r=1)
        tol = 5e-8 if d == 1 else 5e-7
        assert rel_linf(t, ref) <= tol and rel_linf(tt, reft) <= tol, (kernel, rel_linf(t, ref), rel_linf(tt, reft))


def test_r1_divergence_and_w1_sandwich(capi, ctx):
    """Alg. 2 with r = 1 on the c1 inputs (d = 1, n = m = 1000, lam = 20): s~ and s match the
    dense oracle within SPEC's r = 1 gate (1e-6) and s <= W_1 <= s~ with the exact 1-D W_1."""
    from oracle import exact_ot
    cfg = get("c1")
    x, y, a, b = make_inputs(cfg)
    lam, iters, N = 20.0, 200, 256
    ref, _, _ = dense.sinkhorn_divergence(x, y, a, b, lam, iters, r=1)
    P = capi.Plan(ctx, dev(x), dev(y), lam, N, 2.0, 8, 1 / 16, 8, r=1, near_cells=16)
    da, db = dev(a), dev(b)
    u, v, info = capi.sinkhorn_run(P, da, db, iters)
    sd, sc = capi.sinkhorn_divergence(P, da, db, u, v)
    assert abs(sc - ref["s_cost"]) <= 1e-6 * abs(ref["s_cost"]), (sc, ref)
    assert abs(sd - ref["s_dual"]) <= 1e-6 * abs(ref["s_dual"]), (sd, ref)
    W = exact_ot.w1_1d(x[:, 0], a, y[:, 0], b)
    assert sd <= W <= sc


@pytest.mark.parametrize("name,n,m", [("c3", 200000, 200000), ("c5", 400000, 320000)])
def test_pruned_fft_equals_full_fft(capi, ctx, name, n, m):
    """NEXT-4: the box/band-pruned a4-a6 stages (batched 1-D transforms over the rows that can be
    nonzero or are read) equal the full n^3 cuFFT path: a multi-dimensional DFT is the product of
    its 1-D DFTs, and the skipped rows are zero in (outside the box) or discarded (outside the
    band / box)."""
    cfg = get(name)
    x, y, a, b = make_inputs(cfg.with_(n=n, m=m))
    P1 = capi.Plan(ctx, dev(x), dev(y), cfg.lam, cfg.N, cfg.sigma, cfg.m_w, cfg.eps_B, cfg.p)
    os.environ["SK_NO_PRUNED_FFT"] = "1"
    try:
        P0 = capi.Plan(ctx, dev(x), dev(y), cfg.lam, cfg.N, cfg.sigma, cfg.m_w, cfg.eps_B, cfg.p)
    finally:
        del os.environ["SK_NO_PRUNED_FFT"]
    for tr, w in ((0, b), (1, a)):
        for kernel in (0, 1):
            t1 = capi.fastsum_apply(P1, dev(w), tr, kernel).cpu().numpy()
            t0 = capi.fastsum_apply(P0, dev(w), tr, kernel).cpu().numpy()
            assert rel_linf(t1, t0) <= 1e-13, (tr, kernel, rel_linf(t1, t0))


# ------------------------------------------------------------------ degenerate and empty inputs
@pytest.mark.parametrize("d", [1, 2, 3])
def test_degenerate_coincident_points(capi, ctx, d):
    """All atoms of both measures at one point (bbox diagonal 0): K = 1, so pi = a b^T after one
    iteration, s~ = 0 and s = -(H(a) + H(b)) / lam (Eq. (14) with log u_i + log v_j = log a_i +
    log b_j and unit mass). The plan takes the diag -> 0 limit of rho = L / diag (reading Q6b:
    lam' = 1e-16, where the regularised kernel is constant to 1e-21 and its Fourier series exact),
    so the fast summation is exact up to the window error at any N, here lam = 7 and N = 32.
    Tolerance on s: 1e-12 at m_w = 8 (d = 1, 2), 1e-10 at m_w = 6 (d = 3), the Kaiser-Bessel
    window error per mode at sigma = 2 (pins G2/G3: 2.4e-14 / 7.8e-11 per axis)."""
    rng = np.random.default_rng(d)
    n, m, lam = 37, 29, 7.0
    x, y = np.full((n, d), 0.3), np.full((m, d), 0.3)
    a, b = rng.random(n), rng.random(m)
    a, b = a / a.sum(), b / b.sum()
    m_w = 6 if d == 3 else 8
    P = capi.Plan(ctx, dev(x), dev(y), lam, 32, 2.0, m_w)
    centre, rho, _ = nfft_ref.geometry(x, y, 1 / 16, lam)
    assert abs(P.info()["rho"] - rho) <= 1e-15 * rho and abs(P.info()["lambda_p"] - 1e-16) <= 1e-30
    u, v, info = capi.sinkhorn_run(P, dev(a), dev(b), 5)
    sd, sc = capi.sinkhorn_divergence(P, dev(a), dev(b), u, v)
    H = -(a * np.log(a)).sum() - (b * np.log(b)).sum()
    assert abs(sc) <= 1e-15
    assert abs(sd + H / lam) <= (1e-12 if m_w == 8 else 1e-10) * H / lam


def test_empty_measure_is_rejected(capi, ctx):
    """A measure with no atoms at all (every rank empty) has no geometry: SK_EGEOMETRY; a side
    empty while the other is not is a valid plan whose matvec into it is empty."""
    x = np.random.default_rng(0).random((10, 2))
    with pytest.raises(capi.SkError) as e:
        capi.Plan(ctx, dev(np.zeros((0, 2))), dev(np.zeros((0, 2))), 10.0, 32)
    assert e.value.code == capi.SK_EGEOMETRY
    P = capi.Plan(ctx, dev(x), dev(np.zeros((0, 2))), 10.0, 32)
    t = capi.fastsum_apply(P, dev(np.zeros(0)), 0, 0).cpu().numpy()
    assert t.shape == (10,) and np.all(t == 0.0)


def test_short_runs_and_rescale_policies(capi, ctx):
    """iters = 1 and 2 run eagerly (no graph replay): the scalings equal the oracle's Alg. 1
    after the same number of iterations; rescale policy 2 (v <- v / max v, reading Q4) is a pure
    gauge like policy 1."""
    cfg = get("c3").with_(n=3000, m=2500)
    x, y, a, b = make_inputs(cfg)
    a, b = a / a.sum(), b / b.sum()
    P = capi.Plan(ctx, dev(x), dev(y), cfg.lam, cfg.N, cfg.sigma, cfg.m_w, cfg.eps_B, cfg.p)
    for iters in (1, 2):
        u, v, info = capi.sinkhorn_run(P, dev(a), dev(b), iters)
        al, at, bad = dense.sinkhorn_plain(x, y, a, b, cfg.lam, iters)
        assert bad == 0 and info.iters_done == iters
        assert rel_linf(u.cpu().numpy(), al) <= 1e-10 and rel_linf(v.cpu().numpy(), at) <= 1e-10
    s0 = capi.sinkhorn_divergence(P, dev(a), dev(b), *capi.sinkhorn_run(P, dev(a), dev(b), 25)[:2])
    s2 = capi.sinkhorn_divergence(P, dev(a), dev(b), *capi.sinkhorn_run(P, dev(a), dev(b), 25, rescale_policy=2)[:2])
    assert abs(s0[1] - s2[1]) <= 1e-11 * abs(s0[1]) and abs(s0[0] - s2[0]) <= 1e-11 * abs(s0[0])


def test_independent_plans_interleaved(capi, ctx):
    """Two live plans of different sizes (distinct cuFFT handles from the pool, distinct scratch)
    applied alternately give the same results as each alone."""
    c3 = get("c3").with_(n=4000, m=3000)
    c2 = get("c2").with_(n=5000, m=4000)
    x3, y3, a3, b3 = make_inputs(c3)
    x2, y2, a2, b2 = make_inputs(c2)
    P3 = capi.Plan(ctx, dev(x3), dev(y3), c3.lam, c3.N, c3.sigma, c3.m_w, c3.eps_B, c3.p)
    t3 = capi.fastsum_apply(P3, dev(b3), 0, 0).cpu().numpy()
    P2 = capi.Plan(ctx, dev(x2), dev(y2), c2.lam, c2.N, c2.sigma, c2.m_w, c2.eps_B, c2.p)
    t2 = capi.fastsum_apply(P2, dev(b2), 0, 0).cpu().numpy()
    for _ in range(3):
        u3 = capi.fastsum_apply(P3, dev(b3), 0, 0).cpu().numpy()
        u2 = capi.fastsum_apply(P2, dev(b2), 0, 0).cpu().numpy()
        assert rel_linf(u3, t3) <= 1e-13 and rel_linf(u2, t2) <= 1e-13


# ------------------------------------------------------------------ randomized breadth
_RAND_CASES = [(d, seed) for d in (1, 2, 3) for seed in range(4)]


@pytest.mark.parametrize("d,seed", _RAND_CASES)
def test_random_configs_match_method_statement(capi, ctx, d, seed):
    """Seeded random plans (dimension, sizes with ragged tails, lambda, N, m_w, point
    distributions) through every code path the plan may pick (v1 / tiled / DMMA spread and
    interp, x-pair segments, pruned FFT): the GPU fast summation equals the oracle's statement of
    the same method with exact NDFTs (nfft_ref.fastsum_ndft) to the window error, and the direct
    sum to the method error, for both kernels and directions."""
    from oracle import nfft_ref
    rng = np.random.default_rng(1000 * d + seed)
    n, m = int(rng.integers(1, 260)), int(rng.integers(1, 260))
    N = int(rng.choice([16, 24, 32])) if d == 3 else int(rng.choice([16, 32, 48, 64]))
    m_w = int(rng.choice([6, 8])) if 2 * N >= 32 else 6
    lam = float(rng.uniform(5.0, 60.0))
    lo = rng.uniform(-2, 2, size=d)
    span = rng.uniform(0.2, 3.0)
    x = lo + span * rng.random((n, d)) ** float(rng.uniform(0.5, 2.0))   # skewed densities
    y = lo + span * rng.random((m, d))
    wy, wx = rng.random(m), rng.random(n)
    P = capi.Plan(ctx, dev(x), dev(y), lam / span ** 2, N, 2.0, m_w)
    window = 1e-13 if m_w == 8 else 1e-9   # per-mode KB window error at sigma = 2 (G2/G3)
    for kernel in (0, 1):
        t = capi.fastsum_apply(P, dev(wy), 0, kernel).cpu().numpy()
        tt = capi.fastsum_apply(P, dev(wx), 1, kernel).cpu().numpy()
        ref = nfft_ref.fastsum_ndft(x, y, wy, lam / span ** 2, N, 1 / 16, 8, kernel)
        reft = nfft_ref.fastsum_ndft(y, x, wx, lam / span ** 2, N, 1 / 16, 8, kernel)
        assert rel_linf(t, ref) <= window * d and rel_linf(tt, reft) <= window * d, \
            (d, n, m, N, m_w, kernel, rel_linf(t, ref), rel_linf(tt, reft))


@pytest.mark.parametrize("lam,kernel", [(20.0, 0), (20.0, 1), (3000.0, 0), (3000.0, 1)])
def test_r1_d1_nearfield_tiles(capi, ctx, lam, kernel):
    """d = 1 near field at a size spanning many 128-target CTAs, several 256-source blocks per CTA
    (clustered targets: ~400 sources within the radius) and a ragged tail: GPU = the oracle's
    statement of the method. lam = 20 takes the factored exp(-lam'|x - y|) = g_i f_j path,
    lam = 3000 (lam' x span > 600) the per-pair exp."""
    from oracle import laplace_ref as LR
    rng = np.random.default_rng(77)
    n, m = 8000 + 37, 8000 + 13
    x = np.clip(rng.normal(0.5, 0.05, (n, 1)), 0.0, 1.0)
    y = rng.random((m, 1))
    wy, wx = rng.random(m), rng.random(n)
    P = capi.Plan(ctx, dev(x), dev(y), lam, 256, 2.0, 8, 1 / 16, 8, r=1, near_cells=16)
    t = capi.fastsum_apply(P, dev(wy), 0, kernel).cpu().numpy()
    tt = capi.fastsum_apply(P, dev(wx), 1, kernel).cpu().numpy()
    ref = LR.fastsum_ndft(x, y, wy, lam, 256, 1 / 16, 8, 16, kernel=kernel)
    reft = LR.fastsum_ndft(y, x, wx, lam, 256, 1 / 16, 8, 16, kernel=kernel)
    assert rel_linf(t, ref) <= 1e-12 and rel_linf(tt, reft) <= 1e-12, (rel_linf(t, ref), rel_linf(tt, reft))


@pytest.mark.parametrize("d,N,kernel", [(2, 64, 0), (2, 64, 1), (3, 32, 0), (3, 32, 1)])
def test_r1_tiled_nearfield(capi, ctx, d, N, kernel):
    """d >= 2 near field (one CTA per <= 64 targets of a tile, source-tile runs streamed through
    shared memory) at sizes spanning many items and several staged blocks per item, clustered
    targets and a ragged tail: GPU = the oracle's statement of the method."""
    from oracle import laplace_ref as LR
    rng = np.random.default_rng(300 + d)
    n, m = (6000 + 37, 5000 + 11) if d == 2 else (4000 + 37, 3000 + 11)
    x = np.clip(rng.normal(0.5, 0.12, (n, d)), 0.0, 1.0)
    y = rng.random((m, d))
    wy, wx = rng.random(m), rng.random(n)
    m_w = 8 if d == 2 else 6
    P = capi.Plan(ctx, dev(x), dev(y), 20.0, N, 2.0, m_w, 1 / 16, 8, r=1, near_cells=16)
    t = capi.fastsum_apply(P, dev(wy), 0, kernel).cpu().numpy()
    tt = capi.fastsum_apply(P, dev(wx), 1, kernel).cpu().numpy()
    ref = LR.fastsum_ndft(x, y, wy, 20.0, N, 1 / 16, 8, 16, kernel=kernel)
    reft = LR.fastsum_ndft(y, x, wx, 20.0, N, 1 / 16, 8, 16, kernel=kernel)
    window = 1e-12 if d < 3 else 1e-9
    assert rel_linf(t, ref) <= window and rel_linf(tt, reft) <= window, (rel_linf(t, ref), rel_linf(tt, reft))


@pytest.mark.parametrize("d,seed", [(1, 0), (1, 1), (2, 0), (2, 1), (3, 0)])
def test_random_r1_configs_match_method_statement(capi, ctx, d, seed):
    """r = 1 plans with seeded random sizes, lambda, N and near-field radius: GPU = the oracle's
    statement of the method (laplace_ref.fastsum_ndft) to the window error."""
    from oracle import laplace_ref as LR
    rng = np.random.default_rng(2000 + 10 * d + seed)
    n, m = int(rng.integers(1, 200)), int(rng.integers(1, 200))
    N = int(rng.choice([32, 64])) if d < 3 else 32
    near = int(rng.choice([8, 12, 16]))
    lam = float(rng.uniform(5.0, 40.0))
    x, y = rng.random((n, d)), rng.random((m, d))
    wy, wx = rng.random(m), rng.random(n)
    P = capi.Plan(ctx, dev(x), dev(y), lam, N, 2.0, 8 if d < 3 else 6, 1 / 16, 8, r=1, near_cells=near)
    window = 1e-12 if d < 3 else 1e-9
    for kernel in (0, 1):
        t = capi.fastsum_apply(P, dev(wy), 0, kernel).cpu().numpy()
        tt = capi.fastsum_apply(P, dev(wx), 1, kernel).cpu().numpy()
        ref = LR.fastsum_ndft(x, y, wy, lam, N, 1 / 16, 8, near, kernel=kernel)
        reft = LR.fastsum_ndft(y, x, wx, lam, N, 1 / 16, 8, near, kernel=kernel)
        assert rel_linf(t, ref) <= window and rel_linf(tt, reft) <= window, (d, n, m, N, near, kernel)


# ------------------------------------------------------------------ deterministic spread
def _with_env(env, fn):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return fn()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("name", ["c1", "c2", "c5"])
def test_deterministic_spread_is_bitwise_reproducible(capi, ctx, name):
    """SK_DETERMINISTIC=1 (fixed-point box accumulation of the spread, DESIGN.md "Deterministic
    spread"): two back-to-back full-size solves on the same inputs give bit-identical s, s~ and
    scalings (c1 d = 1, c2 d = 2 at kappa 10^10.4, c5 d = 3 at 1e8 + 8e7 nodes), and the results
    match the default atomic mode's to the rounding the conditioning allows."""
    cfg = get(name)
    x, y, a, b = make_inputs(cfg)
    iters = cfg.iters if name != "c5" else 10

    def solve():
        P = capi.Plan(ctx, dev(x), dev(y), cfg.lam, cfg.N, cfg.sigma, cfg.m_w, cfg.eps_B, cfg.p)
        u, v, info = capi.sinkhorn_run(P, dev(a), dev(b), iters)
        sd, sc = capi.sinkhorn_divergence(P, dev(a), dev(b), u, v)
        P.close()
        return sd, sc, u.cpu().numpy(), v.cpu().numpy()

    r1 = _with_env({"SK_DETERMINISTIC": "1"}, solve)
    r2 = _with_env({"SK_DETERMINISTIC": "1"}, solve)
    assert r1[0] == r2[0] and r1[1] == r2[1], (r1[:2], r2[:2])
    assert np.array_equal(r1[2], r2[2]) and np.array_equal(r1[3], r2[3])
    r0 = _with_env({"SK_DETERMINISTIC": "0"}, solve)
    tol = 1e-5 if name == "c2" else 1e-8
    assert abs(r0[1] - r1[1]) <= tol * abs(r0[1]) and abs(r0[0] - r1[0]) <= tol * abs(r0[0]), (r0[:2], r1[:2])


def test_deterministic_spread_properties(capi, ctx):
    """Deterministic spread, stage level: nfft_spread twice gives bit-identical
    grids for every kernel family (d = 1 per-tap, d = 2 DMMA, d = 3 dense / sparse / x-pair TMA
    spreads), equal to the FP64-atomic spread to rounding; weights spanning 1e-30 .. 1e30 keep
    their relative accuracy where they dominate (the scale follows max |w|), all-zero weights
    give an all-zero grid, and a NaN weight gives a non-finite grid instead of a silent number."""
    rng = np.random.default_rng(5)
    for d, N, m_w, cnt in ((1, 64, 8, 500), (2, 32, 8, 3000), (3, 16, 6, 4000)):
        x, y = rng.random((cnt, d)), rng.random((cnt + 5, d))
        mk = lambda: capi.Plan(ctx, dev(x), dev(y), 20.0, N, 2.0, m_w)  # noqa: E731
        Pd = _with_env({"SK_DETERMINISTIC": "1"}, mk)
        Pa = _with_env({"SK_DETERMINISTIC": "0"}, mk)
        Px = _with_env({"SK_DETERMINISTIC": "1", "SK_XPAIRS": "1"}, mk) if d == 3 else None
        for w in (rng.random(cnt), rng.random(cnt) * 10.0 ** rng.uniform(-30, 30, cnt)):
            g1 = capi.nfft_spread(Pd, 0, dev(w)).cpu().numpy()
            g2 = capi.nfft_spread(Pd, 0, dev(w)).cpu().numpy()
            ga = capi.nfft_spread(Pa, 0, dev(w)).cpu().numpy()
            assert np.array_equal(g1, g2), d
            assert np.abs(g1 - ga).max() <= 1e-14 * np.abs(ga).max(), (d, np.abs(g1 - ga).max() / np.abs(ga).max())
            if Px is not None:   # x-pair segments (opt-in)
                gx1 = capi.nfft_spread(Px, 0, dev(w)).cpu().numpy()
                gx2 = capi.nfft_spread(Px, 0, dev(w)).cpu().numpy()
                assert np.array_equal(gx1, gx2)
                assert np.abs(gx1 - ga).max() <= 1e-14 * np.abs(ga).max()
        if Px is not None:
            Px.close()
        assert not np.any(capi.nfft_spread(Pd, 0, dev(np.zeros(cnt))).cpu().numpy())
        wn = rng.random(cnt)
        wn[cnt // 2] = np.nan
        assert not np.all(np.isfinite(capi.nfft_spread(Pd, 0, dev(wn)).cpu().numpy()))
        Pd.close()
        Pa.close()


def test_deterministic_emulated_two_ranks_reproducible(capi):
    """The multi-rank code path (SK_EMULATE_WORLD=2: box exchange, scalar all-reduces, graph
    capture) with the deterministic spread: two solves bit-identical."""
    cfg = get("c3").with_(n=20000, m=15000)
    x, y, a, b = make_inputs(cfg)
    a, b = a / a.sum() / 2, b / b.sum() / 2
    os.environ["SK_EMULATE_WORLD"] = "2"
    try:
        c2 = capi.Context(0)
    finally:
        del os.environ["SK_EMULATE_WORLD"]
    out = []
    for _ in range(2):
        P = capi.Plan(c2, dev(x), dev(y), cfg.lam, cfg.N, cfg.sigma, cfg.m_w, cfg.eps_B, cfg.p)
        u, v, _ = capi.sinkhorn_run(P, dev(a), dev(b), 12)
        out.append((capi.sinkhorn_divergence(P, dev(a), dev(b), u, v), u.cpu().numpy(), v.cpu().numpy()))
        P.close()
    assert out[0][0] == out[1][0] and np.array_equal(out[0][1], out[1][1]) and np.array_equal(out[0][2], out[1][2])
    c2.close()


@pytest.mark.parametrize("N,sigma,det", [(16, 4.0, "1"), (32, 2.0, "1"), (64, 2.0, "0"), (64, 2.0, "1"),
                                         (128, 2.0, "1"), (128, 4.0, "0"), (256, 4.0, "1"), (48, 2.0, "1")])
def test_fftconv2_equals_cufft_path(capi, ctx, N, sigma, det):
    """d = 2 shared-memory FFT convolution (fftconv2.cu: box rows -> band columns x D -> box rows,
    the deterministic conversion fused into the first pass) against the cuFFT D2Z / multiply /
    Z2D path of the same plan (SK_NO_FFTCONV2), both kernels and directions, deterministic and
    atomic spreads, grid edges n = 64 .. 1024 (48 x 2 = 96 is not a power of two: both plans take
    cuFFT); and against the oracle's exact-NDFT statement of the method where it is
    cheap. Clustered x and a narrow y keep the touched box smaller than the grid."""
    rng = np.random.default_rng(N + int(10 * sigma))
    n, m = 3001, 2503
    x = np.concatenate([0.3 + 0.05 * rng.normal(size=(n // 2, 2)), rng.random((n - n // 2, 2))])
    y = 0.2 + 0.6 * rng.random((m, 2)) ** 1.5
    wy, wx = rng.random(m), rng.random(n)
    lam = 0.5 * N
    old = {k: os.environ.get(k) for k in ("SK_DETERMINISTIC", "SK_NO_FFTCONV2")}
    res = {}
    try:
        os.environ["SK_DETERMINISTIC"] = det
        for path in ("fc", "cufft"):
            if path == "cufft":
                os.environ["SK_NO_FFTCONV2"] = "1"
            P = capi.Plan(ctx, dev(x), dev(y), lam, N, sigma, 8)
            res[path] = [capi.fastsum_apply(P, dev(w), tr, k).cpu().numpy()
                         for k in (0, 1) for tr, w in ((0, wy), (1, wx))]
            P.close()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    for i, (a, b) in enumerate(zip(res["fc"], res["cufft"])):
        assert rel_linf(a, b) <= 1e-13, (N, sigma, det, i, rel_linf(a, b))
    if N <= 64:
        for i, (k, tr) in enumerate([(0, 0), (0, 1), (1, 0), (1, 1)]):
            xs, ys, w = (x, y, wy) if tr == 0 else (y, x, wx)
            ref = nfft_ref.fastsum_ndft(xs, ys, w, lam, N, 1 / 16, 8, k)
            assert rel_linf(res["fc"][i], ref) <= 2e-13, (N, sigma, k, tr, rel_linf(res["fc"][i], ref))
