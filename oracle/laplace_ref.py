"""Fast summation for the cost d^r with r = 1 (Laplace kernel exp(-lam |x - y|)), SURVEY §8(f)
NEXT-2. TEST INFRASTRUCTURE. Plain numpy, slow, small cases only.

The paper treats r = 1 in one sentence: "in case of r = 1 we have to regularize the
function K around the point x = 0 in addition ... we add a so called nearfield", and points to
[PlPoStTa18, Sec. 7.5]. Readings:

  geometry      as reading Q6; exp(-lam |x - y|) = exp(-lam' |x' - y'|) with lam' = lam / rho.
  radial_kernel K(r) = exp(-lam' r) (kernel 0); c K with c = r / rho the original distance
                (kernel 1, the integrand of s~ = sum pi d, Def 3.1).
  taylor_KI     inner regularisation on [0, a]: the even polynomial of degree 2p - 2 in r,
                K_I(r) = sum_{i<p} c_i (r/a)^{2i}, with K_I^{(k)}(a) = K^{(k)}(a), k < p (the
                two-point Taylor interpolant of the even extension at -a and a, smooth at 0).
                a = near_cells / (sigma N): the near-field radius in torus units.
  taylor_KB     the boundary regularisation of P:L489-496 with the r = 1 derivatives.
  regularized_kernel  K_R = K_I on |x| <= a, K on (a, L], K_B on (L, 1/2], K_B(1/2) outside.
  bk_sampled    b_k of K_R, exactly as nfft_ref.bk_sampled (2N grid, FFT, centred band).
  fastsum_ndft  Eq. (fastsum) with exact NDFTs for the far field (b_k of K_R) plus the
                near field sum_{|x'_i - y'_j| < a} w_j (K - K_I)(|x'_i - y'_j|), by brute force.
"""
from __future__ import annotations

import math

import numpy as np

from . import nfft_ref


def geometry(x, y, eps_B, lam=None):
    centre, rho, L = nfft_ref.geometry(x, y, eps_B, lam, r=1)
    return centre, rho, L


def radial_derivs(r, lamp, rho, kernel, p):
    """[f^{(k)}(r), k < p] of f(r) = P0(r) exp(-lamp r), P0 = 1 or r / rho; P_{k+1} = P_k' - lamp P_k."""
    P = np.polynomial.Polynomial([1.0]) if kernel == 0 else np.polynomial.Polynomial([0.0, 1.0 / rho])
    e = math.exp(-lamp * r)
    out = []
    for _ in range(p):
        out.append(P(r) * e)
        P = P.deriv() - lamp * P
    return np.array(out)


def radial_kernel(r, lamp, rho, kernel):
    r = np.asarray(r, dtype=np.float64)
    k = np.exp(-lamp * r)
    return k if kernel == 0 else (r / rho) * k


def taylor_KI(lamp, rho, kernel, a, p):
    """c_0..c_{p-1} of K_I(r) = sum_i c_i (r/a)^{2i}: K_I^{(k)}(a) = K^{(k)}(a), k < p."""
    dK = radial_derivs(a, lamp, rho, kernel, p)
    A = np.zeros((p, p))
    rhs = np.zeros(p)
    for k in range(p):
        # d^k/dr^k (r/a)^{2i} at r = a = (2i)! / (2i - k)! / a^k
        for i in range(p):
            e = 2 * i
            if e >= k:
                A[k, i] = math.factorial(e) / math.factorial(e - k) / a ** k
        rhs[k] = dK[k]
    return np.linalg.solve(A, rhs)


def eval_KI(c, r, a):
    t2 = (np.asarray(r, dtype=np.float64) / a) ** 2
    return np.polynomial.polynomial.polyval(t2, c)


def regularized_kernel(xs, lamp, rho, kernel, L, p, a, h=1.0):
    r = np.sqrt((np.asarray(xs) ** 2).sum(axis=-1))
    cI = taylor_KI(lamp, rho, kernel, a, p)
    cB = nfft_ref.taylor_KB(lamp, rho, kernel, L, p, h,
                            derivs=lambda rr, pp: radial_derivs(rr, lamp, rho, kernel, pp))
    return np.where(r <= a, eval_KI(cI, r, a),
                    np.where(r <= L, radial_kernel(r, lamp, rho, kernel),
                             np.where(r <= h / 2, nfft_ref.eval_KB(cB, np.minimum(r, h / 2), L, h),
                                      nfft_ref.eval_KB(cB, h / 2, L, h))))


def bk_sampled(d, N, lamp, rho, kernel, L, p, a):
    M = 2 * N
    g1 = (np.arange(M) - M // 2) / M
    grids = np.meshgrid(*([g1] * d), indexing="ij")
    xs = np.stack(grids, axis=-1)
    Kt = regularized_kernel(xs, lamp, rho, kernel, L, p, a)
    B = np.fft.fftshift(np.fft.fftn(np.fft.ifftshift(Kt)) / M ** d)
    sl = tuple(slice(M // 2 - N // 2, M // 2 + N // 2 + 1) for _ in range(d))
    return B[sl]


def fastsum_ndft(x, y, w, lam, N, eps_B, p, near_cells, sigma=2.0, kernel=0):
    """t_i ~ sum_j w_j K(|x_i - y_j|) for r = 1: NDFT far field of K_R + brute-force near field."""
    x = np.asarray(x, dtype=np.float64).reshape(len(x), -1)
    y = np.asarray(y, dtype=np.float64).reshape(len(y), -1)
    w = np.asarray(w, dtype=np.float64)
    d = x.shape[1]
    centre, rho, L = geometry(x, y, eps_B, lam)
    lamp = lam / rho
    a = near_cells / (sigma * N)
    xs, ys = nfft_ref.scale(x, centre, rho), nfft_ref.scale(y, centre, rho)
    ks, kw = nfft_ref.band(N, d)
    B = bk_sampled(d, N, lamp, rho, kernel, L, p, a).real.reshape(-1)
    far = nfft_ref.ndft_trafo(ks, kw * B * nfft_ref.ndft_adjoint(ks, ys, w), xs).real
    cI = taylor_KI(lamp, rho, kernel, a, p)
    near = np.zeros(x.shape[0])
    for i in range(x.shape[0]):
        r = np.sqrt(((ys - xs[i]) ** 2).sum(axis=1))
        m = r < a
        if m.any():
            near[i] = np.sum(w[m] * (radial_kernel(r[m], lamp, rho, kernel) - eval_KI(cI, r[m], a)))
    return far + near
