"""Convergence diagnostics of Sinkhorn's iteration (Sec. 3.3). TEST INFRASTRUCTURE.

  sinkhorn_trace  Alg. 1 in the scaling domain with the dense kernel matrix
                  k_ij = exp(-lambda |x_i - y_j|^2) (Eq. (MatrixK_sin_div)), alpha^0 =
                  alpha~^0 = 1, odd Delta first. Before every half-step it records
                  the residual of the marginal that the half-step makes exact (Eq. (Error)
                  P:L333-336) and its Kullback-Leibler divergence D_KL(p | pi 1) (definition at
                  P:L322, the quantity of the Lemma at); after it, sum p log alpha.
                  Columns as sinkhorn_run_trace in include/sinkhorn_nfft.h.
  objective       f(alpha, alpha~) of Eq. (objfunc) with the unnormalised k.
  iteration_bound 2 eps^-2 log(kappa / jmath) of the Theorem at, kappa = sum of
                  the entries of pi, jmath = min_ij k~_ij with k~ = k / ||k||_1.

Dense O(n m) memory: small cases only (n, m <= a few thousand).
"""
from __future__ import annotations

import numpy as np

FIELDS = ("row_resid", "row_kl", "sum_a_log_u", "col_resid", "col_kl", "sum_b_log_v")


def kernel_matrix(x, y, lam):
    x = np.asarray(x, dtype=np.float64).reshape(len(x), -1)
    y = np.asarray(y, dtype=np.float64).reshape(len(y), -1)
    c = ((x[:, None, :] - y[None, :, :]) ** 2).sum(-1)
    return np.exp(-lam * c)


def _kl(p, q):
    m = p > 0
    return float(np.sum(p[m] * np.log(p[m] / q[m])))


def sinkhorn_trace(x, y, a, b, lam, iters, history=False):
    """Returns (trace [iters, 6], alpha, alpha~[, [(alpha, alpha~) after every half-step]])."""
    k = kernel_matrix(x, y, lam)
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    al, at = np.ones(k.shape[0]), np.ones(k.shape[1])
    tr = np.empty((iters, 6))
    hist = []
    for it in range(iters):
        # odd Delta (Eq. (even_sin_div)): alpha <- p / (k alpha~)
        kv = k @ at
        row = al * kv                                   # pi^Delta 1 before the update
        tr[it, 0] = np.abs(row - a).sum()
        tr[it, 1] = _kl(a, row)
        al = a / kv
        tr[it, 2] = float(np.sum(a * np.log(al)))
        if history:
            hist.append((al.copy(), at.copy()))
        # even Delta (Eq. (odd_sin_div)): alpha~ <- p~ / (k^T alpha)
        ku = k.T @ al
        col = at * ku
        tr[it, 3] = np.abs(col - b).sum()
        tr[it, 4] = _kl(b, col)
        at = b / ku
        tr[it, 5] = float(np.sum(b * np.log(at)))
        if history:
            hist.append((al.copy(), at.copy()))
    return (tr, al, at, hist) if history else (tr, al, at)


def objective(k, a, b, al, at):
    """Eq. (objfunc): sum_ij alpha_i k_ij alpha~_j - sum p log alpha - sum p~ log alpha~."""
    return float(al @ (k @ at) - np.sum(a * np.log(al)) - np.sum(b * np.log(at)))


def iteration_bound(k, eps, kappa=1.0):
    """Theorem P:L420-424: Delta* <= 2 eps^-2 log(kappa / jmath), jmath = min k / sum k."""
    jmath = float(k.min() / k.sum())
    return 2.0 / eps ** 2 * np.log(kappa / jmath)
