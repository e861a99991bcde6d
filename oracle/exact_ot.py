"""Exact optimal transport on tiny inputs and the 1-D closed form. TEST INFRASTRUCTURE.

  lp_permutations  Eq. (Da)-(Dd) for n = m <= 8 and uniform weights: the
                   transport polytope's vertices are permutation matrices / n (Birkhoff),
                   so W = min_sigma (1/n) sum_i c_{i sigma(i)}.
  lp_linprog       Eq. (Da)-(Dd) for general weights with scipy's HiGHS LP solver as the
                   library step.
  w1_1d            d = 1, cost |x - y| (r = 1, NEXT-2): W_1 = int |F - G| ds.
  w2_1d            d = 1, cost |x - y|^2: W_2^2 = int_0^1 |F^-1(t) - G^-1(t)|^2 dt
                   (BJ north_star), evaluated exactly by merging the quantile step functions.
"""
from __future__ import annotations

import itertools

import numpy as np
from scipy.optimize import linprog


def cost_matrix(x, y, r=2):
    """d_ij^r, d the Euclidean distance; r = 2 or 1."""
    x = np.asarray(x).reshape(len(x), -1)
    y = np.asarray(y).reshape(len(y), -1)
    c = ((x[:, None, :] - y[None, :, :]) ** 2).sum(-1)
    return c if r == 2 else np.sqrt(c)


def lp_permutations(x, y, r=2):
    C = cost_matrix(x, y, r)
    n = C.shape[0]
    assert C.shape[1] == n and n <= 8
    best = np.inf
    for perm in itertools.permutations(range(n)):
        v = C[np.arange(n), perm].sum() / n
        best = min(best, v)
    return best


def lp_linprog(x, y, a, b, r=2):
    C = cost_matrix(x, y, r)
    n, m = C.shape
    A_eq = np.zeros((n + m, n * m))
    for i in range(n):
        A_eq[i, i * m:(i + 1) * m] = 1.0
    for j in range(m):
        A_eq[n + j, j::m] = 1.0
    b_eq = np.concatenate([a, b])
    res = linprog(C.reshape(-1), A_eq=A_eq, b_eq=b_eq, bounds=(0, None), method="highs")
    assert res.success, res.message
    return float(res.fun), res.x.reshape(n, m)


def w1_1d(x, a, y, b):
    """d = 1, cost |x - y| (r = 1): W_1 = int |F(s) - G(s)| ds, F, G the distribution functions
    (the 1-D closed form of the r = 1 transport problem), exact for discrete measures."""
    x = np.asarray(x, dtype=np.float64).reshape(-1)
    y = np.asarray(y, dtype=np.float64).reshape(-1)
    pts = np.concatenate([x, y])
    mass = np.concatenate([np.asarray(a, dtype=np.float64), -np.asarray(b, dtype=np.float64)])
    o = np.argsort(pts, kind="stable")
    pts, mass = pts[o], mass[o]
    diff = np.cumsum(mass)[:-1]              # F - G on each gap between consecutive support points
    return float(np.sum(np.abs(diff) * np.diff(pts)))


def w2_1d(x, a, y, b):
    """int_0^1 |F^{-1}(t) - G^{-1}(t)|^2 dt for discrete measures on R."""
    x = np.asarray(x).reshape(-1)
    y = np.asarray(y).reshape(-1)
    ix, iy = np.argsort(x, kind="stable"), np.argsort(y, kind="stable")
    xs, as_ = x[ix], np.asarray(a)[ix]
    ys, bs = y[iy], np.asarray(b)[iy]
    Fa = np.cumsum(as_)
    Fb = np.cumsum(bs)
    Fa[-1] = 1.0
    Fb[-1] = 1.0
    cuts = np.unique(np.concatenate([[0.0], Fa, Fb]))
    total = 0.0
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        if hi <= lo:
            continue
        mid = 0.5 * (lo + hi)
        qa = xs[min(np.searchsorted(Fa, mid), len(xs) - 1)]
        qb = ys[min(np.searchsorted(Fb, mid), len(ys) - 1)]
        total += (hi - lo) * (qa - qb) ** 2
    return total
