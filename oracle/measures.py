"""Entropy and KL divergence (Lemma 3.2; §3.4). TEST INFRASTRUCTURE."""
from __future__ import annotations

import numpy as np


def entropy(p):
    """H(P) = -sum p_i log p_i (natural log), zero weights contribute 0."""
    p = np.asarray(p, dtype=np.float64)
    q = p[p > 0]
    return float(-(q * np.log(q)).sum())


def kl(p, q):
    """D_KL(p | q) = sum p_i log(p_i / q_i)."""
    p = np.asarray(p, dtype=np.float64)
    q = np.asarray(q, dtype=np.float64)
    mask = p > 0
    return float((p[mask] * np.log(p[mask] / q[mask])).sum())
