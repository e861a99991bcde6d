"""Pins of oracle/diagnostics.py (convergence diagnostics) against what
Sec. 3.3 of the paper proves, independently of the trace's own bookkeeping:
  - Lemma: f(alpha^D) - f(alpha^{D+1}) = D_KL(p|pi^D 1) + D_KL(p~|pi^D^T 1), with f
    evaluated from the iterates by Eq. (objfunc) directly (dense k, oracle.diagnostics.objective);
  - Pinsker: ||pi 1 - p||_1 <= sqrt(2 D_KL(p | pi 1)) once pi has unit mass;
  - Theorem: the first D with ||E^D||_1 <= eps satisfies D <= 2 eps^-2 log(kappa/jmath);
  - the trace's final scalings equal the C oracle's Alg. 1 (dense.sinkhorn_plain).
"""
import numpy as np
import pytest

from oracle import dense, diagnostics as D
from synthetic import get, make_inputs


@pytest.fixture(scope="module")
def case():
    cfg = get("c1")
    x, y, a, b = make_inputs(cfg)
    x, y, a, b = x[:400], y[:300], a[:400] / a[:400].sum(), b[:300] / b[:300].sum()
    lam = 30.0
    tr, al, at, hist = D.sinkhorn_trace(x, y, a, b, lam, 25, history=True)
    return x, y, a, b, lam, tr, al, at, hist


def test_lemma_objective_decrease_equals_kl(case):
    x, y, a, b, lam, tr, al, at, hist = case
    k = D.kernel_matrix(x, y, lam)
    f = [D.objective(k, a, b, u, v) for u, v in hist]        # after half-steps 1, 2, ...
    kl = []                                                  # KL before half-steps 2, 3, ...
    for it in range(tr.shape[0]):
        if it > 0:
            kl.append(tr[it, 1])
        kl.append(tr[it, 4])
    for dlt in range(len(f) - 1):
        assert abs((f[dlt] - f[dlt + 1]) - kl[dlt]) <= 1e-12 * max(1.0, abs(f[dlt])), dlt
    assert all(np.diff(f) <= 1e-15)


def test_pinsker_after_first_half_step(case):
    """Checked while D_KL is far above its FP64 evaluation error (sum p log(p/q) with q ~ p
    cancels to ~1e-16 absolute)."""
    *_, tr, al, at, hist = case
    checked = 0
    for it in range(tr.shape[0]):
        for r, k in ((0, 1), (3, 4)):
            if (it > 0 or r == 3) and tr[it, k] > 1e-10:
                assert tr[it, r] <= np.sqrt(2 * tr[it, k]) * (1 + 1e-6)
                checked += 1
    assert checked >= 10


def test_iteration_bound(case):
    x, y, a, b, lam, tr, al, at, hist = case
    k = D.kernel_matrix(x, y, lam)
    E = []                                  # ||E^D||_1 for D = 1, 2, ...: before each half-step
    for it in range(tr.shape[0]):
        E += [tr[it, 0], tr[it, 3]]
    E = E[1:]                               # D = 0 is the unscaled k (not a coupling)
    for eps in (0.3, 0.1, 0.03, 0.01):
        first = next(d + 1 for d, e in enumerate(E) if e <= eps)
        assert first <= D.iteration_bound(k, eps)


def test_trace_scalings_match_c_oracle(case):
    x, y, a, b, lam, tr, al, at, hist = case
    al2, at2, bad = dense.sinkhorn_plain(x, y, a, b, lam, tr.shape[0])
    assert bad == 0
    assert np.abs(al2 / al - 1).max() < 1e-13 and np.abs(at2 / at - 1).max() < 1e-13
    assert abs(tr[-1, 2] - np.sum(a * np.log(al2))) < 1e-12 * abs(tr[-1, 2])
