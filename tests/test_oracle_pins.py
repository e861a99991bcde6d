"""Pins of the CPU oracle to what the paper and mathematics fix (no GPU).

Every oracle function is checked against something other than itself: closed forms
printed in / derived from the paper, brute force, an independent library routine, or
high-precision arithmetic. Each test names the pin id of DESIGN.md "Oracle pins".
"""
import itertools
import json
import math
import os

import mpmath
import numpy as np
import pytest
from scipy import integrate

from oracle import dense, exact_ot, measures, nfft_ref
from synthetic import get, make_inputs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _load_golden(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


# ---------------------------------------------------------------- P1: 2x2 closed form
def test_P1_two_point_closed_form():
    """x = y = {0,1}, a = b = (1/2,1/2), lam = 1 (golden/p1_two_point.json).
    By symmetry alpha = alpha~ = t, t^2 (1 + e^-1) = 1/2 (Eq. (S1)):
    s~ = e^-1/(1+e^-1), s = log t^2 = -log(2(1+e^-1))."""
    gd = _load_golden("p1_two_point.json")
    x = np.array([[0.0], [1.0]])
    a = np.array([0.5, 0.5])
    res, f, g = dense.sinkhorn_divergence(x, x, a, a, 1.0, 50)
    assert abs(res["s_cost"] - gd["s_cost"]) < 1e-15
    assert abs(res["s_dual"] - gd["s_dual"]) < 1e-15
    # high-precision fixed point of Eq. (S1) reproduces the same numbers
    mpmath.mp.dps = 50
    t2 = mpmath.mpf(1) / (2 * (1 + mpmath.e ** -1))
    assert abs(float(2 * t2 * mpmath.e ** -1) - res["s_cost"]) < 1e-15
    assert abs(float(mpmath.log(t2)) - res["s_dual"]) < 1e-15
    # plain-domain Alg. 1 agrees with the log-domain iterates
    al, at, bad = dense.sinkhorn_plain(x, x, a, a, 1.0, 50)
    assert bad == 0
    np.testing.assert_allclose(np.log(al) + np.log(at[0]), (f + g[0]) * 1.0, atol=1e-14)


# ---------------------------------------------------------------- P2: n = 1
def test_P2_single_source_atom():
    """n = 1: pi_1j = b_j after the first v-update, so s~ = sum_j b_j c(x1, y_j) and
    s = s~ - H(b)/lam (Def 3.1)."""
    rng = np.random.default_rng(1)
    x = rng.random((1, 2))
    y = rng.random((7, 2))
    b = rng.random(7)
    b /= b.sum()
    lam = 3.0
    res, _, _ = dense.sinkhorn_divergence(x, y, np.array([1.0]), b, lam, 3)
    c = ((x - y) ** 2).sum(1)
    s_cost = float((b * c).sum())
    assert abs(res["s_cost"] - s_cost) < 1e-15
    assert abs(res["s_dual"] - (s_cost - measures.entropy(b) / lam)) < 1e-14


# ---------------------------------------------------------------- P3: LP sandwich
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_P3_lp_sandwich_and_limit(seed):
    """s <= W <= s~, s~ - W <= (H(pi^s) - H(pi^W))/lam (Lemma 3.2 P:L152-160,
    Prop 3.3); s~ -> W as lam grows. W by brute force over permutations
    (Birkhoff), cross-checked against an LP solve."""
    rng = np.random.default_rng(seed)
    n = 6
    x, y = rng.random((n, 2)), rng.random((n, 2))
    a = np.full(n, 1.0 / n)
    W = exact_ot.lp_permutations(x, y)
    W_lp, plan = exact_ot.lp_linprog(x, y, a, a)
    assert abs(W - W_lp) < 1e-12
    H_W = measures.entropy(plan.reshape(-1))
    prev = None
    for lam in [2.0, 5.0, 10.0, 20.0]:
        res, _, _ = dense.sinkhorn_divergence(x, y, a, a, lam, 20000)
        assert res["col_resid"] < 1e-12 and res["row_resid"] < 1e-10
        assert res["s_dual"] <= W + 1e-12
        assert W <= res["s_cost"] + 1e-12
        assert res["s_cost"] - W <= (res["entropy"] - H_W) / lam + 1e-10
        assert W - res["s_dual"] <= res["entropy"] / lam + 1e-10
        gap = res["s_cost"] - W
        if prev is not None:
            assert gap <= prev + 1e-12
        prev = gap
    # lam -> infinity: s~ -> W (checked with a long run at lam = 100 where the iteration
    # still converges; the gap is O(1/lam) and must shrink by >= 4x for 5x lam)
    res, _, _ = dense.sinkhorn_divergence(x, y, a, a, 100.0, 100000)
    assert abs(res["s_cost"] - W) < 0.25 * prev


def test_P3_lp_general_weights_vs_sinkhorn_limit():
    """General weights: transportation LP (HiGHS) vs the Sinkhorn upper divergence at
    large lam, on a 1-D instance where W is also given by the quantile closed form."""
    rng = np.random.default_rng(7)
    x, y = rng.random(5), rng.random(4)
    a, b = rng.random(5) + 0.1, rng.random(4) + 0.1
    a, b = a / a.sum(), b / b.sum()
    W_lp, _ = exact_ot.lp_linprog(x, y, a, b)
    W_q = exact_ot.w2_1d(x, a, y, b)
    assert abs(W_lp - W_q) < 1e-12
    res, _, _ = dense.sinkhorn_divergence(x[:, None], y[:, None], a, b, 2000.0, 20000)
    assert res["s_dual"] <= W_lp + 1e-12 <= res["s_cost"] + 2e-12
    assert res["s_cost"] - W_lp < 5e-3


# ---------------------------------------------------------------- P4: 1-D closed form
@pytest.mark.parametrize("seed", range(4))
def test_P4_w2_1d_equals_lp(seed):
    """W_2^2 = int |F^-1 - G^-1|^2 (BJ north_star) equals the LP optimum on random 1-D
    instances; translation by c gives c^2; W(P,P) = 0."""
    rng = np.random.default_rng(100 + seed)
    n, m = rng.integers(2, 9, size=2)
    x, y = rng.normal(size=n), rng.normal(size=m)
    a, b = rng.random(n) + 0.05, rng.random(m) + 0.05
    a, b = a / a.sum(), b / b.sum()
    W_lp, _ = exact_ot.lp_linprog(x, y, a, b)
    assert abs(exact_ot.w2_1d(x, a, y, b) - W_lp) < 1e-12
    assert abs(exact_ot.w2_1d(x, a, x + 0.3, a) - 0.09) < 1e-14
    assert exact_ot.w2_1d(x, a, x, a) == 0.0


def test_P4_sinkhorn_tends_to_w2_1d():
    """Sinkhorn upper divergence tends to the 1-D closed form as lam grows (O(1/lam))."""
    rng = np.random.default_rng(3)
    x, y = rng.random(40), rng.random(40) * 0.5 + 0.3
    a = np.full(40, 1 / 40)
    W = exact_ot.w2_1d(x, a, y, a)
    errs = []
    for lam in [100.0, 1000.0, 10000.0]:
        res, _, _ = dense.sinkhorn_divergence(x[:, None], y[:, None], a, a, lam, 20000)
        errs.append(abs(res["s_cost"] - W))
        assert res["s_dual"] <= W + 1e-12 <= res["s_cost"] + 1e-12
    assert errs[2] < errs[1] < errs[0] and errs[2] < 1e-3


# ---------------------------------------------------------------- P5/P6: marginals, identical
def test_P5_marginals_and_P6_identical_symmetric():
    """Column marginal exact after each v-update, row residual -> 0 (Eq. (Error));
    identical measures: s(P,P) <= 0 <= s~(P,P) <= (H(pi^s) - H(P))/lam (Prop 3.3 with W = 0,
    H(pi^W) = H(P)); symmetry s(P,Q) = s(Q,P) at convergence."""
    cfg = get("c1")
    x, y, a, b = make_inputs(cfg)
    x, y, a, b = x[:300], y[:300], a[:300] * 1000 / 300, b[:300] * 1000 / 300
    lam = 30.0
    r_prev = None
    for T in [5, 20, 80]:
        res, _, _ = dense.sinkhorn_divergence(x, y, a, b, lam, T)
        assert res["col_resid"] < 1e-14
        if r_prev is not None:
            assert res["row_resid"] < r_prev
        r_prev = res["row_resid"]
    assert r_prev < 1e-6
    pp, _, _ = dense.sinkhorn_divergence(x, x, a, a, lam, 200)
    assert pp["s_dual"] <= 0.0 <= pp["s_cost"]
    assert pp["s_cost"] <= (pp["entropy"] - measures.entropy(a)) / lam + 1e-12
    pq, _, _ = dense.sinkhorn_divergence(x, y, a, b, lam, 300)
    qp, _, _ = dense.sinkhorn_divergence(y, x, b, a, lam, 300)
    assert abs(pq["s_dual"] - qp["s_dual"]) < 1e-12
    assert abs(pq["s_cost"] - qp["s_cost"]) < 1e-12
    # s~ - s = H(pi)/lam at convergence (Def 3.1)
    assert abs(pq["s_cost"] - pq["s_dual"] - pq["entropy"] / lam) < 1e-10


# ---------------------------------------------------------------- O1 direct sum pins
def test_O1_direct_sum_lattice_separable():
    """Pin G4: on a common K x K lattice the Gaussian sum is separable and Toeplitz
    (P:L471-472): t = A V A^T, A_pq = exp(-lam (p-q)^2 / K^2); for c exp(-lam c):
    t_c = A_c V A^T + A V A_c^T with A_c = ((p - q)/K)^2 A."""
    K, lam = 24, 40.0
    i = np.arange(K) / K
    gx, gy = np.meshgrid(i, i, indexing="ij")
    pts = np.stack([gx.ravel(), gy.ravel()], 1)
    V = np.random.default_rng(5).random((K, K))
    dq = (i[:, None] - i[None, :]) ** 2
    A = np.exp(-lam * dq)
    Ac = dq * A
    t0 = dense.direct_sum(pts, pts, V.ravel(), lam, 0).reshape(K, K)
    t1 = dense.direct_sum(pts, pts, V.ravel(), lam, 1).reshape(K, K)
    np.testing.assert_allclose(t0, A @ V @ A.T, rtol=1e-13)
    np.testing.assert_allclose(t1, Ac @ V @ A.T + A @ V @ Ac.T, rtol=1e-12)


def test_O1_direct_sum_highprecision_rows_and_adjointness():
    """A few rows at 40 digits (mpmath) and <u, K v> = <K^T u, v> with rows subset."""
    rng = np.random.default_rng(11)
    x, y = rng.random((50, 3)), rng.random((60, 3))
    w, u = rng.random(60), rng.random(50)
    lam = 20.0
    t = dense.direct_sum(x, y, w, lam, 0)
    tc = dense.direct_sum(x, y, w, lam, 1)
    mpmath.mp.dps = 40
    for i in [0, 17, 49]:
        s = mpmath.fsum(mpmath.mpf(w[j]) * mpmath.exp(-lam * mpmath.fsum((mpmath.mpf(x[i, a]) - y[j, a]) ** 2 for a in range(3))) for j in range(60))
        sc = mpmath.fsum(mpmath.mpf(w[j]) * mpmath.fsum((mpmath.mpf(x[i, a]) - y[j, a]) ** 2 for a in range(3))
                         * mpmath.exp(-lam * mpmath.fsum((mpmath.mpf(x[i, a]) - y[j, a]) ** 2 for a in range(3))) for j in range(60))
        assert abs(float(s) - t[i]) <= 2e-16 * abs(float(s))
        assert abs(float(sc) - tc[i]) <= 2e-16 * abs(float(sc))
    tT = dense.direct_sum(y, x, u, lam, 0)
    assert abs(u @ t - tT @ w) < 1e-14 * abs(u @ t)
    rows = np.array([3, 40, 7])
    np.testing.assert_array_equal(dense.direct_sum(x, y, w, lam, 0, rows=rows), t[rows])


# ---------------------------------------------------------------- window / NDFT / NFFT pins
@pytest.mark.parametrize("m,sigma", [(6, 2.0), (8, 2.0)])
def test_window_transform_pair(m, sigma):
    """Fourier transform of the Kaiser-Bessel window by quadrature equals the I0 closed form
    used for the deconvolution (reading Q10)."""
    n = 128
    for k in [0, 5, 17, 32]:
        xi = k / n
        val, _ = integrate.quad(lambda u: nfft_ref.kb_phi(np.array([u]), m, sigma)[0] * math.cos(2 * math.pi * xi * u),
                                -m, m, limit=400, epsabs=0, epsrel=1e-13)
        ref = nfft_ref.kb_phihat(k, n, m, sigma)
        assert abs(val - ref) < 1e-11 * ref


def test_ndft_equispaced_is_fft():
    """On equispaced nodes j/M the adjoint NDFT is the DFT (numpy FFT as library step)."""
    M, N = 16, 8
    nodes = (np.arange(M) / M)[:, None]
    w = np.random.default_rng(2).random(M)
    ks, _ = nfft_ref.band(N, 1)
    a = nfft_ref.ndft_adjoint(ks, nodes, w)
    F = np.fft.fft(w)
    np.testing.assert_allclose(a, F[ks[:, 0].astype(int) % M], rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(nfft_ref.ndft_adjoint(ks, np.zeros((1, 1)), [1.0]), 1.0)


@pytest.mark.parametrize("d,m,tol", [(1, 8, 5e-14), (2, 8, 5e-14), (1, 6, 5e-10), (2, 6, 5e-10)])
def test_gridding_plus_fft_is_ndft(d, m, tol):
    """NFFT identity: spread (grid_spread) + FFT + division by prod phihat reproduces the
    adjoint NDFT on the band to the window error; interpolation of the NDFT-synthesised
    grid reproduces ndft_trafo."""
    N, sigma = 16, 2.0
    n = int(sigma * N)
    rng = np.random.default_rng(d * 10 + m)
    pts = (rng.random((40, d)) - 0.5) * 0.45
    w = rng.random(40)
    g = nfft_ref.grid_spread(pts, w, n, m, sigma)
    G = np.fft.fftn(g)
    ks, _ = nfft_ref.band(N, d)
    idx = tuple((ks[:, a].astype(int)) % n for a in range(d))
    # grid index l <-> position l/n - 1/2: undo the half shift with (-1)^{sum k}
    shift = (-1.0) ** ks.sum(1)
    ph = np.prod([nfft_ref.kb_phihat(ks[:, a], n, m, sigma) for a in range(d)], axis=0)
    approx = G[idx] * shift / ph
    exact = nfft_ref.ndft_adjoint(ks, pts, w)
    assert np.abs(approx - exact).max() <= tol * np.abs(exact).max()
    # trafo: t(x) = sum_k fhat_k e^{2 pi i k x}
    fhat = rng.normal(size=len(ks)) + 1j * rng.normal(size=len(ks))
    H = np.zeros((n,) * d, dtype=complex)
    H[idx] = fhat * shift / ph
    Hg = np.fft.ifftn(H) * n ** d
    t_re = nfft_ref.grid_interp(Hg.real, pts, m, sigma) + 1j * nfft_ref.grid_interp(Hg.imag, pts, m, sigma)
    t_ex = nfft_ref.ndft_trafo(ks, fhat, pts)
    assert np.abs(t_re - t_ex).max() <= tol * np.abs(fhat).sum()


# ---------------------------------------------------------------- kernel coefficient pins
def test_taylor_KB_interpolation_conditions():
    """K_B^{(k)}(L) = K^{(k)}(L), k < p and K_B^{(k)}(1/2) = 0, 1 <= k < p (Eq. intpol_cond_3/4),
    derivatives of K by mpmath numerical differentiation (independent of the recursion)."""
    lamp, rho, L, p = 3.0, 1.3, 0.5 - 1 / 16, 8
    mpmath.mp.dps = 40
    for kernel in (0, 1):
        c = nfft_ref.taylor_KB(lamp, rho, kernel, L, p)
        D = 0.5 - L
        P = np.polynomial.Polynomial(c)
        f = (lambda r: mpmath.exp(-lamp * r * r)) if kernel == 0 else (lambda r: r * r / rho ** 2 * mpmath.exp(-lamp * r * r))
        for k in range(p):
            dk = float(mpmath.diff(f, mpmath.mpf(L), k))
            got = P.deriv(k)(0.0) / D ** k if k else P(0.0)
            assert abs(got - dk) <= 1e-10 * max(1.0, abs(dk))
        for k in range(1, p):
            # roundoff bound of evaluating the k-th derivative of sum c_i t^i at t = 1
            scale = sum(abs(ci) * math.perm(i, k) for i, ci in enumerate(c) if i >= k)
            assert abs(P.deriv(k)(1.0)) <= 1e-13 * scale


@pytest.mark.parametrize("cfg_name", ["c1", "c2", "c3", "c5"])
def test_G1_bk_sampled_matches_closed_form(cfg_name):
    """b_k from sampled K~_per (2N grid, FFT, truncate; reading Q9) equals the closed-form
    periodised-Gaussian coefficients to ~1e-15 b_0 (K_B is inert: K(L) <= e^-60)."""
    cfg = get(cfg_name)
    d = cfg.d
    N = min(cfg.N, 64)
    # geometry of the unit cube: diag = sqrt(d)
    L = 0.5 - cfg.eps_B
    rho = L / math.sqrt(d)
    lamp = cfg.lam / rho ** 2
    for kernel in (0, 1):
        Bs = nfft_ref.bk_sampled(d, N, lamp, rho, kernel, L, cfg.p)
        Bg = nfft_ref.bk_gauss(d, N, lamp, rho, kernel)
        scale = np.abs(Bg).max()
        assert np.abs(Bs - Bg).max() <= 2e-15 * scale * (4 if d == 3 else 1)


def test_fastsum_ndft_matches_direct_sum():
    """Eq. (fastsum) with exact NDFTs and truncation at the stated N reproduces the direct
    sum (Eq. (matexp)) to the Fourier truncation level exp(-pi^2 (N/2)^2 / lam')."""
    rng = np.random.default_rng(4)
    x, y = rng.random((30, 2)), rng.random((25, 2))
    w = rng.random(25)
    # lam' = lam / rho^2 = 313: K(L) = e^-60 (K_B inert, as in every BJ config) and the
    # Fourier truncation exp(-pi^2 (N/2)^2 / lam') = e^-32 at N = 64
    lam, N = 30.0, 64
    for kernel in (0, 1):
        t_dir = dense.direct_sum(x, y, w, lam, kernel)
        t_nd = nfft_ref.fastsum_ndft(x, y, w, lam, N, 1 / 16, 8, kernel)
        assert np.abs(t_nd - t_dir).max() < 1e-12 * np.abs(t_dir).max()


def test_geometry_reading():
    """Q6: scaled nodes lie in |x'| <= L/2, pairwise |x'-y'| <= L, and the kernel is
    invariant: exp(-lam |x-y|^2) = exp(-lam' |x'-y'|^2)."""
    rng = np.random.default_rng(9)
    x, y = rng.random((100, 3)) * 3 - 1, rng.random((80, 3))
    c, rho, L = nfft_ref.geometry(x, y, 1 / 16)
    xs, ys = nfft_ref.scale(x, c, rho), nfft_ref.scale(y, c, rho)
    assert np.sqrt((xs ** 2).sum(1)).max() <= L / 2 * (1 + 1e-15)
    assert np.sqrt((ys ** 2).sum(1)).max() <= L / 2 * (1 + 1e-15)
    D2 = ((x[:, None] - y[None]) ** 2).sum(-1)
    D2s = ((xs[:, None] - ys[None]) ** 2).sum(-1)
    np.testing.assert_allclose(np.exp(-2.0 * D2), np.exp(-2.0 / rho ** 2 * D2s), rtol=1e-13)


# ---------------------------------------------------------------- measures
def test_measures_examples():
    """SPEC S:L55-67 examples (entropy, KL) by direct arithmetic."""
    assert abs(measures.entropy([0.25] * 4) - math.log(4)) < 1e-15
    assert abs(measures.entropy([0.5, 0.25, 0.25]) - 1.5 * math.log(2)) < 1e-15
    assert abs(measures.kl([0.75, 0.25], [0.5, 0.5]) - (0.75 * math.log(1.5) + 0.25 * math.log(0.5))) < 1e-15
    assert measures.kl([0.5, 0.5], [0.5, 0.5]) == 0.0


# ---------------------------------------------------------------- Alg. 2 on the method's fast summation
@pytest.mark.parametrize("d,N", [(1, 32), (2, 16), (3, 12)])
def test_fastsum_operator_matches_fastsum_ndft(d, N):
    """FastsumOperator (axis-separable NDFTs) equals fastsum_ndft (one dense band x node phase
    matrix, pinned against the direct sum above) for both kernels and directions."""
    rng = np.random.default_rng(20 + d)
    x, y = rng.random((37, d)), rng.random((41, d))
    w, wx = rng.random(41), rng.random(37)
    op = nfft_ref.FastsumOperator(x, y, 20.0, N, 1 / 16, 8)
    for k in (0, 1):
        ref = nfft_ref.fastsum_ndft(x, y, w, 20.0, N, 1 / 16, 8, k)
        reft = nfft_ref.fastsum_ndft(y, x, wx, 20.0, N, 1 / 16, 8, k)
        assert np.abs(op.apply(w, False, k) - ref).max() <= 1e-14 * np.abs(ref).max()
        assert np.abs(op.apply(wx, True, k) - reft).max() <= 1e-14 * np.abs(reft).max()


def test_sinkhorn_fastsum_equals_dense_when_resolved_and_not_otherwise():
    """Alg. 2 on the method's operator (nfft_ref.sinkhorn_fastsum) equals the dense log-domain
    Alg. 1 when the band resolves the kernel (c1 inputs, N = 96: truncation e^-43), and differs
    from it when it does not (N = 40: the c exp(-lam c) kernel is truncated at ~e^-9), so the
    function really runs the truncated method and not the exact kernel."""
    cfg = get("c1")
    x, y, a, b = make_inputs(cfg)
    x, y, a, b = x[:300], y[:300], a[:300] / a[:300].sum(), b[:300] / b[:300].sum()
    ref, _, _ = dense.sinkhorn_divergence(x, y, a, b, cfg.lam, 60)
    good = nfft_ref.sinkhorn_fastsum(x, y, a, b, cfg.lam, 96, cfg.eps_B, cfg.p, 60)
    assert abs(good["s_cost"] - ref["s_cost"]) <= 1e-9 * ref["s_cost"]
    assert abs(good["s_dual"] - ref["s_dual"]) <= 1e-9 * abs(ref["s_dual"])
    # the scalings are Alg. 1's: column marginal exact after the v-update
    op = nfft_ref.FastsumOperator(x, y, cfg.lam, 96, cfg.eps_B, cfg.p)
    col = good["alpha_t"] * op.apply(good["alpha"], True, 0)
    assert np.abs(col - b).max() <= 1e-14
    bad = nfft_ref.sinkhorn_fastsum(x, y, a, b, cfg.lam, 40, cfg.eps_B, cfg.p, 60)
    assert abs(bad["s_cost"] - ref["s_cost"]) >= 1e-6 * ref["s_cost"]


@pytest.mark.parametrize("d", [1, 2, 3])
def test_degenerate_geometry_limit(d):
    """Reading Q6b: all atoms at one point (diag = 0). The plan takes the limit diag -> 0 of
    rho = L / diag (lam' = 1e-16), where K is constant: the fast summation returns sum_j w_j for
    K and 0 for c K (c = 0) to rounding at any N, and Alg. 2 gives s~ = 0, s = -(H(a)+H(b))/lam."""
    x, y = np.full((5, d), 0.3), np.full((4, d), 0.3)
    w = np.random.default_rng(d).random(4)
    c, rho, L = nfft_ref.geometry(x, y, 1 / 16, 7.0)
    assert abs(7.0 / rho ** 2 - nfft_ref.LAMP_DEGENERATE) <= 1e-30
    for N in (16, 32):
        t0 = nfft_ref.fastsum_ndft(x, y, w, 7.0, N, 1 / 16, 8, 0)
        t1 = nfft_ref.fastsum_ndft(x, y, w, 7.0, N, 1 / 16, 8, 1)
        assert np.abs(t0 - w.sum()).max() <= 4e-16 * w.sum() and np.abs(t1).max() <= 1e-20
    a, b = np.full(5, 0.2), np.full(4, 0.25)
    r = nfft_ref.sinkhorn_fastsum(x, y, a, b, 7.0, 16, 1 / 16, 8, 3)
    assert abs(r["s_cost"]) <= 1e-20
    assert abs(r["s_dual"] + (math.log(5) + math.log(4)) / 7.0) <= 1e-15


@pytest.mark.parametrize("d,N,m,tol", [(1, 32, 8, 5e-14), (2, 16, 8, 5e-14), (3, 12, 6, 2e-11), (3, 16, 8, 1e-13)])
def test_nfft_operator_is_ndft_operator_to_window_error(d, N, m, tol):
    """NfftFastsumOperator (gridding with the window matrix + FFT + phihat deconvolution)
    equals FastsumOperator (exact NDFTs) to the Kaiser-Bessel window error at sigma = 2 (pins G2/G3),
    and its window matrix equals the dense gridding definition grid_spread."""
    rng = np.random.default_rng(30 + d + m)
    x, y = rng.random((37, d)), rng.random((41, d))
    w, wx = rng.random(41), rng.random(37)
    op = nfft_ref.FastsumOperator(x, y, 20.0, N, 1 / 16, 8)
    opn = nfft_ref.NfftFastsumOperator(x, y, 20.0, N, 1 / 16, 8, m, 2.0)
    for k in (0, 1):
        ref, reft = op.apply(w, False, k), op.apply(wx, True, k)
        assert np.abs(opn.apply(w, False, k) - ref).max() <= tol * np.abs(ref).max()
        assert np.abs(opn.apply(wx, True, k) - reft).max() <= tol * np.abs(reft).max()
    c, rho, _ = nfft_ref.geometry(x, y, 1 / 16, 20.0)
    ys = nfft_ref.scale(y, c, rho)
    g = nfft_ref.grid_spread(ys, w, 2 * N, m, 2.0).ravel()
    assert np.abs(nfft_ref.window_matrix(ys, 2 * N, m, 2.0).T @ w - g).max() <= 1e-15 * np.abs(g).max()
