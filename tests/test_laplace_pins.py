"""Pins of the r = 1 oracle (cost |x - y|, Laplace kernel exp(-lam |x - y|)),
against closed forms, exact LP, independent matrix routes and mpmath (no retyped formulas)."""
import math

import mpmath
import numpy as np
import pytest

from oracle import dense, exact_ot, laplace_ref as LR
from synthetic import get, make_inputs


def test_direct_sum_r1_lattice_toeplitz():
    """1-D lattice x = y = k/K: the r = 1 kernel matrix is Toeplitz A_pq = exp(-lam |p - q|/K);
    the direct sum equals A @ w (independent route)."""
    K, lam = 257, 13.0
    x = (np.arange(K) / K)[:, None]
    w = np.random.default_rng(0).random(K)
    p = np.arange(K)
    A = np.exp(-lam * np.abs(p[:, None] - p[None, :]) / K)
    for kernel, M in ((0, A), (1, A * np.abs(p[:, None] - p[None, :]) / K)):
        t = dense.direct_sum(x, x, w, lam, kernel, r=1)
        assert np.abs(t - M @ w).max() <= 1e-14 * np.abs(M @ w).max()


def test_radial_derivs_r1_mpmath():
    lamp, rho, r = 37.0, 0.3, 0.021
    for kernel in (0, 1):
        f = (lambda s: mpmath.exp(-lamp * s)) if kernel == 0 else (lambda s: s / rho * mpmath.exp(-lamp * s))
        got = LR.radial_derivs(r, lamp, rho, kernel, 8)
        for k in range(8):
            ref = float(mpmath.diff(f, r, k))
            assert abs(got[k] - ref) <= 1e-12 * max(1.0, abs(ref)), (kernel, k)


@pytest.mark.parametrize("p", [4, 6, 8])
def test_inner_regularisation_conditions(p):
    """K_I matches K and its first p - 1 derivatives at r = a (mpmath differentiation of the
    returned polynomial) and is even (K_I'(0) = 0)."""
    lamp, rho, a = 80.0, 0.4, 1 / 32
    for kernel in (0, 1):
        c = LR.taylor_KI(lamp, rho, kernel, a, p)
        poly = lambda s: sum(mpmath.mpf(ci) * (s / a) ** (2 * i) for i, ci in enumerate(c))
        dK = LR.radial_derivs(a, lamp, rho, kernel, p)
        for k in range(p):
            got = float(mpmath.diff(poly, mpmath.mpf(a), k))
            assert abs(got - dK[k]) <= 1e-9 * max(abs(dK[k]), abs(dK[0]) / a ** k), (kernel, k)
        assert abs(float(mpmath.diff(poly, mpmath.mpf(0), 1))) == 0.0


@pytest.mark.parametrize("d,n", [(1, 300), (2, 150)])
def test_fastsum_r1_matches_direct_sum(d, n):
    """Far field (NDFT of K_R) + near field reproduces the r = 1 direct sum to the method error
    (N = 128, near field 16 cells, p = 8: ~1e-8 in 1-D, ~1e-7 in 2-D here; SPEC's r = 1 gate
    is 1e-6)."""
    rng = np.random.default_rng(d)
    x, y = rng.random((n, d)), rng.random((n + 7, d))
    w = rng.random(n + 7)
    for lam in (20.0, 50.0):
        ref = dense.direct_sum(x, y, w, lam, 0, r=1)
        t = LR.fastsum_ndft(x, y, w, lam, 128, 1 / 16, 8, 16)
        assert np.abs(t - ref).max() <= (5e-8 if d == 1 else 5e-7) * np.abs(ref).max(), (d, lam)


def test_w1_closed_form_equals_lp():
    rng = np.random.default_rng(5)
    for _ in range(5):
        x, y = rng.random(7), rng.random(6)
        a, b = rng.random(7), rng.random(6)
        a, b = a / a.sum(), b / b.sum()
        lp, _ = exact_ot.lp_linprog(x, y, a, b, r=1)
        assert abs(exact_ot.w1_1d(x, a, y, b) - lp) <= 1e-12


def test_sinkhorn_r1_sandwich_and_limit():
    """Prop. 3.3 sandwich s <= W_1 <= s~ with the exact LP, and s~ -> W_1 as lam grows."""
    rng = np.random.default_rng(7)
    x, y = rng.random((6, 2)), rng.random((6, 2))
    a = np.full(6, 1 / 6)
    W = exact_ot.lp_permutations(x, y, r=1)
    gaps = []
    for lam in (5.0, 50.0, 500.0):
        ref, _, _ = dense.sinkhorn_divergence(x, y, a, a, lam, 3000, r=1)
        assert ref["s_dual"] <= W + 1e-12 <= ref["s_cost"] + 2e-12
        gaps.append(ref["s_cost"] - W)
    assert gaps[0] > gaps[1] > gaps[2] and gaps[2] < 1e-3


def test_single_source_r1_closed_form():
    """n = 1: pi_1j = b_j, so s~ = sum_j b_j |x_1 - y_j| (pin P2 with r = 1)."""
    rng = np.random.default_rng(2)
    x, y = rng.random((1, 2)), rng.random((9, 2))
    b = rng.random(9)
    b /= b.sum()
    ref, _, _ = dense.sinkhorn_divergence(x, y, np.ones(1), b, 10.0, 3, r=1)
    assert abs(ref["s_cost"] - float((b * np.sqrt(((x - y) ** 2).sum(1))).sum())) <= 1e-14
