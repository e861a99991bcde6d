"""Plain numpy reference of the fast-summation building blocks. TEST INFRASTRUCTURE.

Each function is a direct (slow) statement of one definition from PAPER.md §4
 under the readings listed in DESIGN.md "Readings of the paper":

  geometry       Q6: torus period h = 1, L = 1/2 - eps_B, nodes scaled into the ball
                 |x'| <= L/2 about the bbox midpoint, rho = L / diag(bbox(x u y)),
                 lam' = lam / rho^2 so that exp(-lam |x - y|^2) = exp(-lam' |x' - y'|^2)
                 ("we assume that we have |x_j| <= L/2, i.e. |x_i - x~_j| <= L").
  kb_phi         Q10: Kaiser-Bessel window of the NFFT ("window function with
                 small support"), in oversampled-grid units u:
                   phi(u) = sinh(beta sqrt(m^2 - u^2)) / (pi sqrt(m^2 - u^2)),  |u| < m,
                 beta = pi (2 - 1/sigma), 0 for |u| > m (beta/pi at |u| = m).
  kb_phihat      its continuous Fourier transform  int phi(u) e^{-2 pi i xi u} du
                   = I0(m sqrt(beta^2 - (2 pi xi)^2)),  xi = k / (sigma N).
  ndft_adjoint   inner sum of Eq. (fastsum): a_k = sum_j w_j e^{-2 pi i k.y_j}
  ndft_trafo     outer sum: t_i = sum_k fhat_k e^{2 pi i k.x_i}
  radial_kernel  K(r) = exp(-lam' r^2) (kernel 0) and c(r) K(r), c = r^2 / rho^2 (kernel 1)
  taylor_KB      two-point Taylor regularisation K_B on [L, h/2]  (Eq. intpol_cond_3/4,
                 P:L489-496): K_B^{(k)}(L) = K^{(k)}(L), k < p; K_B^{(k)}(h/2) = 0, 1 <= k < p.
  regularized_kernel  K~: K on |x|<=L, K_B on (L, h/2], K_B(h/2) outside.
  bk_sampled     b_k of K~_per: sample K~ on a (2N)^d grid of the period cell, FFT, keep
                 the centred N-band (reading Q9).
  bk_gauss       closed form of the Fourier coefficients of the periodised Gaussian (pin G1).
  grid_spread    adjoint-NFFT gridding g[l] = sum_j w_j prod_a phi(n (y_ja + 1/2) - l_a)
  grid_interp    NFFT interpolation  t_i = sum_l G[l] prod_a phi(n (x_ia + 1/2) - l_a)
                 ("s(x) = sum_l s_l phi(x - l/2N)"); grid index l <-> torus
                 position l/n - 1/2, n = sigma N.
  fastsum_ndft   Eq. (fastsum) with exact NDFTs in place of the NFFTs:
                 t_i = sum_{k in band} w_k b_k a_k e^{2 pi i k.x_i}, band {-N/2..N/2}^d with
                 weight 1/2 on each |k_a| = N/2 (reading Q8).
"""
from __future__ import annotations

import itertools
import math

import numpy as np
from scipy import special


# ----------------------------------------------------------------------------- geometry
LAMP_DEGENERATE = 1e-16


def geometry(x, y, eps_B, lam=None, r=2):
    """Return (centre, rho, L). Reading Q6 of P:L479-486.

    Degenerate geometry (every atom at one point, diag = 0; reading Q6b): any rho
    keeps the nodes in the ball, and as diag -> 0 the rule rho = L / diag sends lam' to 0, where
    the kernel is constant and its Fourier series exact. The limit is taken at a finite point:
    rho such that lam' = LAMP_DEGENERATE (lam / rho^2 for r = 2, lam / rho for r = 1), which needs
    lam; without lam (no kernel involved) rho = 1."""
    pts = np.concatenate([np.asarray(x).reshape(len(x), -1), np.asarray(y).reshape(len(y), -1)])
    lo, hi = pts.min(axis=0), pts.max(axis=0)
    centre = 0.5 * (lo + hi)
    diag = float(np.sqrt(((hi - lo) ** 2).sum()))
    L = 0.5 - eps_B
    if diag > 0:
        rho = L / diag
    elif lam is None:
        rho = 1.0
    else:
        rho = math.sqrt(lam / LAMP_DEGENERATE) if r == 2 else lam / LAMP_DEGENERATE
    return centre, rho, L


def scale(pts, centre, rho):
    return rho * (np.asarray(pts).reshape(len(pts), -1) - centre)


# ----------------------------------------------------------------------------- window
def kb_beta(sigma):
    return math.pi * (2.0 - 1.0 / sigma)


def kb_phi(u, m, sigma):
    """Kaiser-Bessel window in grid units (vectorised)."""
    u = np.asarray(u, dtype=np.float64)
    beta = kb_beta(sigma)
    s2 = m * m - u * u
    out = np.zeros_like(u)
    inside = s2 > 0
    s = np.sqrt(s2[inside])
    out[inside] = np.sinh(beta * s) / (math.pi * s)
    out[s2 == 0] = beta / math.pi
    return out


def kb_phihat(k, n, m, sigma):
    """I0(m sqrt(beta^2 - (2 pi k / n)^2)) -- Fourier transform of kb_phi at xi = k/n."""
    beta = kb_beta(sigma)
    k = np.asarray(k, dtype=np.float64)
    return special.i0(m * np.sqrt(beta ** 2 - (2 * math.pi * k / n) ** 2))


# ----------------------------------------------------------------------------- NDFT
def band(N, d):
    """Centred frequency set {-N/2..N/2}^d and the Q8 weights (1/2 on each |k_a| = N/2)."""
    k1 = np.arange(-N // 2, N // 2 + 1)
    w1 = np.where(np.abs(k1) == N // 2, 0.5, 1.0)
    ks = np.array(list(itertools.product(k1, repeat=d)), dtype=np.float64)
    ws = np.array([np.prod(c) for c in itertools.product(w1, repeat=d)])
    return ks, ws


def ndft_adjoint(ks, pts, w):
    """a_k = sum_j w_j exp(-2 pi i k . y_j)  (inner sum of Eq. (fastsum))."""
    ph = np.exp(-2j * math.pi * (ks @ np.asarray(pts).T))
    return ph @ np.asarray(w)


def ndft_trafo(ks, fhat, pts):
    """t_i = sum_k fhat_k exp(2 pi i k . x_i)."""
    ph = np.exp(2j * math.pi * (np.asarray(pts) @ ks.T))
    return ph @ fhat


# ----------------------------------------------------------------------------- kernel
def _radial_derivs(r, lamp, rho, kernel, p):
    """[f^{(k)}(r) for k < p] of f(r) = P0(r) exp(-lamp r^2), P0 = 1 (kernel 0) or r^2/rho^2
    (kernel 1); recursion P_{k+1} = P_k' - 2 lamp r P_k."""
    P = np.polynomial.Polynomial([1.0]) if kernel == 0 else np.polynomial.Polynomial([0, 0, 1.0 / rho ** 2])
    two_lr = np.polynomial.Polynomial([0.0, 2.0 * lamp])
    out = []
    e = math.exp(-lamp * r * r)
    for _ in range(p):
        out.append(P(r) * e)
        P = P.deriv() - two_lr * P
    return np.array(out)


def radial_kernel(r, lamp, rho, kernel):
    r = np.asarray(r, dtype=np.float64)
    k = np.exp(-lamp * r * r)
    return k if kernel == 0 else (r * r / rho ** 2) * k


def taylor_KB(lamp, rho, kernel, L, p, h=1.0, derivs=None):
    """Coefficients c of K_B(r) = sum_i c_i t^i, t = (r - L)/(h/2 - L), degree 2p - 2,
    solving the 2p - 1 interpolation conditions (intpol_cond_3/4).
    derivs(r, p): [K^{(k)}(r), k < p] of the radial profile (default: the r = 2 kernels)."""
    D = h / 2 - L
    deg = 2 * p - 2
    nc = deg + 1
    A = np.zeros((nc, nc))
    rhs = np.zeros(nc)
    dK = derivs(L, p) if derivs is not None else _radial_derivs(L, lamp, rho, kernel, p)
    row = 0
    # d^k/dr^k at r = L (t = 0): k! c_k / D^k = K^{(k)}(L)
    for k in range(p):
        A[row, k] = math.factorial(k) / D ** k
        rhs[row] = dK[k]
        row += 1
    # d^k/dr^k at r = h/2 (t = 1) vanish for k = 1..p-1
    for k in range(1, p):
        for i in range(k, nc):
            A[row, i] = math.factorial(i) / math.factorial(i - k) / D ** k
        row += 1
    return np.linalg.solve(A, rhs)


def eval_KB(c, r, L, h=1.0):
    t = (np.asarray(r) - L) / (h / 2 - L)
    return np.polynomial.polynomial.polyval(t, c)


def regularized_kernel(xs, lamp, rho, kernel, L, p, h=1.0):
    """K~(x) for points xs in the period cell [-h/2, h/2)^d."""
    r = np.sqrt((np.asarray(xs) ** 2).sum(axis=-1))
    c = taylor_KB(lamp, rho, kernel, L, p, h)
    out = np.where(r <= L, radial_kernel(r, lamp, rho, kernel),
                   np.where(r <= h / 2, eval_KB(c, np.minimum(r, h / 2), L, h), eval_KB(c, h / 2, L, h)))
    return out


def bk_sampled(d, N, lamp, rho, kernel, L, p):
    """b_k, k in {-N/2..N/2}^d (as a dense (N+1)^d array, axis index k + N/2), from K~_per
    sampled on the M = 2N grid of [-1/2, 1/2)^d, numpy FFT / M^d (reading Q9)."""
    M = 2 * N
    g1 = (np.arange(M) - M // 2) / M        # positions -1/2 .. 1/2 - 1/M
    grids = np.meshgrid(*([g1] * d), indexing="ij")
    xs = np.stack(grids, axis=-1)
    Kt = regularized_kernel(xs, lamp, rho, kernel, L, p)
    # sample index s <-> position (s - M/2)/M: b_k = (1/M^d) sum_s K(x_s) e^{-2 pi i k x_s}
    B = np.fft.fftn(np.fft.ifftshift(Kt)) / M ** d
    B = np.fft.fftshift(B)                 # axis index k + M/2
    sl = tuple(slice(M // 2 - N // 2, M // 2 + N // 2 + 1) for _ in range(d))
    return B[sl]


def bk_gauss(d, N, lamp, rho, kernel):
    """Closed-form Fourier coefficients of the periodised kernel (pin G1):
    kernel 0: prod_a sqrt(pi/lam') exp(-pi^2 k_a^2 / lam');
    kernel 1: (1/rho^2) sum_a g2(k_a) prod_{a' != a} g0(k_a'),
              g2(k) = sqrt(pi/lam') exp(-pi^2 k^2/lam') (1/(2 lam') - pi^2 k^2 / lam'^2)."""
    k1 = np.arange(-N // 2, N // 2 + 1, dtype=np.float64)
    g0 = np.sqrt(math.pi / lamp) * np.exp(-math.pi ** 2 * k1 ** 2 / lamp)
    g2 = g0 * (1.0 / (2 * lamp) - math.pi ** 2 * k1 ** 2 / lamp ** 2)
    if kernel == 0:
        out = g0
        for _ in range(d - 1):
            out = np.multiply.outer(out, g0)
        return out
    total = 0.0
    for a in range(d):
        term = None
        for ax in range(d):
            f = g2 if ax == a else g0
            term = f if term is None else np.multiply.outer(term, f)
        total = total + term
    return total / rho ** 2


# ----------------------------------------------------------------------------- gridding
def grid_spread(pts_scaled, w, n, m, sigma):
    """g[l] = sum_j w_j prod_a phi(n (y_ja + 1/2) - l_a), l in {0..n-1}^d (dense, small n)."""
    pts = np.asarray(pts_scaled)
    d = pts.shape[1]
    g = np.zeros((n,) * d)
    ls = np.arange(n, dtype=np.float64)
    for j in range(pts.shape[0]):
        u = n * (pts[j] + 0.5)
        f = [kb_phi(u[a] - ls, m, sigma) for a in range(d)]
        t = w[j] * f[0]
        for a in range(1, d):
            t = np.multiply.outer(t, f[a])
        g += t
    return g


def grid_interp(G, pts_scaled, m, sigma):
    """t_i = sum_l G[l] prod_a phi(n (x_ia + 1/2) - l_a)."""
    pts = np.asarray(pts_scaled)
    d = pts.shape[1]
    n = G.shape[0]
    ls = np.arange(n, dtype=np.float64)
    out = np.empty(pts.shape[0])
    for i in range(pts.shape[0]):
        u = n * (pts[i] + 0.5)
        t = G
        for a in range(d):
            t = np.tensordot(kb_phi(u[a] - ls, m, sigma), t, axes=([0], [0]))
        out[i] = float(t)
    return out


# ----------------------------------------------------------------------------- fast summation (NDFT)
def fastsum_ndft(x, y, w, lam, N, eps_B, p, kernel=0, use_closed_form=False):
    """Eq. (fastsum) with exact NDFTs: returns t at the nodes x (original
    coordinates), sources y with weights w. b_k from the sampled K~ unless use_closed_form."""
    x = np.asarray(x).reshape(len(x), -1)
    y = np.asarray(y).reshape(len(y), -1)
    d = x.shape[1]
    centre, rho, L = geometry(x, y, eps_B, lam)
    lamp = lam / rho ** 2
    xs, ys = scale(x, centre, rho), scale(y, centre, rho)
    ks, kw = band(N, d)
    B = bk_gauss(d, N, lamp, rho, kernel) if use_closed_form else bk_sampled(d, N, lamp, rho, kernel, L, p).real
    bflat = B.reshape(-1)          # same itertools.product ordering as band()
    ahat = ndft_adjoint(ks, ys, w)
    return ndft_trafo(ks, kw * bflat * ahat, xs).real


# ----------------------------------------------------------------------------- Alg. 2 on the method's operator
def _axis_phases(pts, N):
    """Per-axis NDFT phases E_a[i, k] = exp(2 pi i k x_ia), k = -N/2 .. N/2 (axis index k + N/2)."""
    k1 = np.arange(-N // 2, N // 2 + 1, dtype=np.float64)
    return [np.exp(2j * math.pi * np.outer(pts[:, a], k1)) for a in range(pts.shape[1])]


class FastsumOperator:
    """The fast summation of Eq. (fastsum) with exact NDFTs, as a reusable linear
    operator on fixed node sets (the matrix-free form of fastsum_ndft):

        (K~ w)_i = sum_{k in band} kw_k b_k a_k(w) e^{2 pi i k.x'_i},
        a_k(w)   = sum_j w_j e^{-2 pi i k.y'_j},

    band and weights kw of reading Q8, b_k = bk_sampled (reading Q9) for kernel 0 (exp(-lam c))
    and kernel 1 (c exp(-lam c)); the transpose swaps the roles of x and y. The d-dimensional
    NDFT is evaluated axis by axis (e^{2 pi i k.x} = prod_a e^{2 pi i k_a x_a}), so the cost is
    O(n (N+1)^d) per product without an (N+1)^d x n phase matrix. Used by sinkhorn_fastsum."""

    def __init__(self, x, y, lam, N, eps_B, p):
        x = np.asarray(x, dtype=np.float64).reshape(len(x), -1)
        y = np.asarray(y, dtype=np.float64).reshape(len(y), -1)
        self.d = d = x.shape[1]
        centre, rho, L = geometry(x, y, eps_B, lam)
        lamp = lam / rho ** 2
        self.Ex = _axis_phases(scale(x, centre, rho), N)
        self.Ey = _axis_phases(scale(y, centre, rho), N)
        k1 = np.arange(-N // 2, N // 2 + 1)
        w1 = np.where(np.abs(k1) == N // 2, 0.5, 1.0)
        kw = w1
        for _ in range(d - 1):
            kw = np.multiply.outer(kw, w1)
        self.coef = [kw * bk_sampled(d, N, lamp, rho, kern, L, p).real for kern in (0, 1)]
        self.N = N

    @staticmethod
    def _adjoint(E, w):
        """a_k = sum_j w_j conj(prod_a E_a[j, k_a]) as an (N+1)^d array."""
        Ec = [e.conj() for e in E]
        if len(E) == 1:
            return Ec[0].T @ w
        if len(E) == 2:
            return (Ec[0] * w[:, None]).T @ Ec[1]
        K = Ec[0].shape[1]
        yz = (Ec[1][:, :, None] * Ec[2][:, None, :]).reshape(-1, K * K)
        return ((Ec[0] * w[:, None]).T @ yz).reshape(K, K, K)

    @staticmethod
    def _trafo(E, F):
        """t_i = Re sum_k F_k prod_a E_a[i, k_a]."""
        if len(E) == 1:
            return (E[0] @ F).real
        if len(E) == 2:
            return ((E[0] @ F) * E[1]).sum(axis=1).real
        K = E[0].shape[1]
        G = (E[0] @ F.reshape(K, K * K)).reshape(-1, K, K)
        return np.einsum("ibc,ib,ic->i", G, E[1], E[2]).real

    def apply(self, w, transpose=False, kernel=0):
        """transpose False: t = K~ w (w on y, t on x); True: t = K~^T w (w on x, t on y)."""
        src, dst = (self.Ex, self.Ey) if transpose else (self.Ey, self.Ex)
        w = np.asarray(w, dtype=np.float64)
        return self._trafo(dst, self.coef[kernel] * self._adjoint(src, w))


def sinkhorn_fastsum(x, y, a, b, lam, N, eps_B, p, iters, window=None):
    """Alg. 2 with the method's own fast summation (FastsumOperator: Eq. (fastsum)
    with exact NDFTs, i.e. the NFFT fast summation without the window error), in the plain
    (scaling) domain exactly as Alg. 2 states it: alpha~ = 1, then per iteration
    alpha = p / (K~ alpha~) (odd Delta, Eq. (even_F_sink)) and
    alpha~ = p~ / (K~^T alpha) (even Delta, Eq. (odd_F_sink)). Returns
    dict(s_dual, s_cost, alpha, alpha_t, min_t) with
      s_dual = (1/lam)(1 + sum p log alpha + sum p~ log alpha~ - sum_j (K~^T alpha)_j alpha~_j)
               (Eq. (14), the Alg. 2 result line P:L732),
      s_cost = sum_i alpha_i ((c K)~ alpha~)_i  (s~ of Def 3.1 P:L137 through the c exp(-lam c)
               fast summation).
    This is the statement of the method whose only error against the dense Alg. 1 is the
    regularised kernel's Fourier truncation and FP64 rounding of the sums: it isolates the
    method's error from an implementation's (SURVEY.md §8(c) consequence (1)).
    window=(m_w, sigma): use NfftFastsumOperator instead -- the complete method with the NFFT's
    window error, i.e. what a faithful implementation computes up to FP64 rounding."""
    op = FastsumOperator(x, y, lam, N, eps_B, p) if window is None else \
        NfftFastsumOperator(x, y, lam, N, eps_B, p, window[0], window[1])
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    al, at = np.ones(a.shape[0]), np.ones(b.shape[0])
    min_t = np.inf
    for _ in range(iters):
        t = op.apply(at, False, 0)
        min_t = min(min_t, float(t.min()))
        al = a / t
        tt = op.apply(al, True, 0)
        min_t = min(min_t, float(tt.min()))
        at = b / tt
    S3 = float(op.apply(al, True, 0) @ at)
    s_dual = (1.0 + float(a @ np.log(al)) + float(b @ np.log(at)) - S3) / lam
    s_cost = float(al @ op.apply(at, False, 1))
    return dict(s_dual=s_dual, s_cost=s_cost, alpha=al, alpha_t=at, min_t=min_t)


def window_matrix(pts_scaled, n, m, sigma):
    """Sparse Phi[j, l] = prod_a phi(n (x_ja + 1/2) - l_a) over the 2m taps per axis
    l_a = floor(u_a) - m + 1 .. floor(u_a) + m (u = n (x + 1/2)); row-major flat grid index.
    The gridding definition of grid_spread / grid_interp as a matrix: g = Phi^T w, t = Phi G
    (P:L475-477)."""
    from scipy import sparse
    pts = np.asarray(pts_scaled, dtype=np.float64)
    cnt, d = pts.shape
    u = n * (pts + 0.5)
    base = np.floor(u).astype(np.int64) - m + 1
    taps = np.arange(2 * m)
    vals = np.ones((cnt, 1))
    flat = np.zeros((cnt, 1), dtype=np.int64)
    for a in range(d):
        la = base[:, a:a + 1] + taps[None, :]                    # [cnt, 2m]
        pa = kb_phi(u[:, a:a + 1] - la, m, sigma)
        vals = (vals[:, :, None] * pa[:, None, :]).reshape(cnt, -1)
        flat = (flat[:, :, None] * n + (la % n)[:, None, :]).reshape(cnt, -1)
    rows = np.repeat(np.arange(cnt), vals.shape[1])
    return sparse.csr_matrix((vals.ravel(), (rows, flat.ravel())), shape=(cnt, n ** d))


class NfftFastsumOperator:
    """The fast summation exactly as the paper builds it (P:L473-477 + Eq. (fastsum)):
    adjoint NFFT of the sources (gridding with the Kaiser-Bessel window on the sigma N grid,
    FFT, division by phihat on the N-band), multiplication by kw_k b_k, NFFT to the targets
    (division by phihat, inverse FFT, window interpolation). The window error is included, so
    an implementation of the method matches this up to FP64 rounding."""

    def __init__(self, x, y, lam, N, eps_B, p, m, sigma):
        x = np.asarray(x, dtype=np.float64).reshape(len(x), -1)
        y = np.asarray(y, dtype=np.float64).reshape(len(y), -1)
        self.d = d = x.shape[1]
        centre, rho, L = geometry(x, y, eps_B, lam)
        lamp = lam / rho ** 2
        self.n = n = int(round(sigma * N))
        self.Phx = window_matrix(scale(x, centre, rho), n, m, sigma)
        self.Phy = window_matrix(scale(y, centre, rho), n, m, sigma)
        ks, kw = band(N, d)
        self.idx = tuple(ks[:, a].astype(int) % n for a in range(d))
        shift = (-1.0) ** ks.sum(1)          # grid index l <-> position l/n - 1/2
        ph = np.prod([kb_phihat(ks[:, a], n, m, sigma) for a in range(d)], axis=0)
        self.deconv = shift / ph
        self.coef = [kw * bk_sampled(d, N, lamp, rho, kern, L, p).real.reshape(-1) for kern in (0, 1)]

    def apply(self, w, transpose=False, kernel=0):
        src, dst = (self.Phx, self.Phy) if transpose else (self.Phy, self.Phx)
        shape = (self.n,) * self.d
        g = (src.T @ np.asarray(w, dtype=np.float64)).reshape(shape)
        ahat = np.fft.fftn(g)[self.idx] * self.deconv                 # adjoint NFFT on the band
        H = np.zeros(shape, dtype=complex)
        H[self.idx] = self.coef[kernel] * ahat * self.deconv
        G = (np.fft.ifftn(H) * self.n ** self.d).real                 # NFFT: grid values
        return dst @ G.ravel()
