"""Write tests/golden/method_envelope.json: what Alg. 2 itself reaches on the conditioning cases,
computed by the oracle only (SURVEY.md §8(c) consequence (1): "parity failures on c1 (at
N = 64), c2 and c4 are properties of Alg. 2 at those inputs").

For each case, on the same seeded inputs:
  dense   oracle.dense.sinkhorn_divergence: log-domain Alg. 1 with exact sums;
          the exact answer up to FP64 rounding, which dense sums keep relative per entry.
  method  oracle.nfft_ref.sinkhorn_fastsum: Alg. 2 with the method's own fast
          summation (Eq. (fastsum) P:L622-631 with exact NDFTs, i.e. without the window error).
          Its distance to `dense` is the method's error at these inputs (Fourier truncation, and
          FP64 rounding of an absolute-error summation amplified by kappa = ||v||_1 / min (K v)).
  nfft    the same with the complete NFFT fast summation (Kaiser-Bessel window, m_w, sigma:
          NfftFastsumOperator): what a faithful implementation computes. nfft and method differ
          only by the window error (~5e-15 per matvec at m_w = 8); their distance at the end of
          Alg. 2 is the spread that FP64-level matvec perturbations cause at these inputs.
  log10_kappa  from the method run: log10(max(||v||_1 / min K v, ||u||_1 / min K^T u)) at the end.

Cases: c1 at BJ's N = 64 and at N = 96; c2 and c4 on their seeded 3000-point subsamples
(synthetic.small_subsample) at lam in LAMS (the BJ lambda is one of them).

    nice python tools/make_golden_method.py
"""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import dense, nfft_ref  # noqa: E402
from synthetic import get, make_inputs, small_subsample  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "method_envelope.json")
K_SUB = 3000
LAMS = {"c2": [5.0, 10.0, 20.0, 50.0, 100.0, 200.0], "c4": [5.0, 10.0, 20.0, 50.0, 100.0, 200.0]}


def kappa_log10(x, y, a, b, lam, N, cfg, iters):
    op = nfft_ref.FastsumOperator(x, y, lam, N, cfg.eps_B, cfg.p)
    r = nfft_ref.sinkhorn_fastsum(x, y, a, b, lam, N, cfg.eps_B, cfg.p, iters)
    al, at = r["alpha"], r["alpha_t"]
    tv = op.apply(at, False, 0)
    kv = math.log10(at.sum() / tv.min()) if tv.min() > 0 else float("inf")
    tu = op.apply(al, True, 0)
    ku = math.log10(al.sum() / tu.min()) if tu.min() > 0 else float("inf")
    return r, max(kv, ku)


def case(name, cfg, x, y, a, b, lam, N):
    t0 = time.time()
    ref, _, _ = dense.sinkhorn_divergence(x, y, a, b, lam, cfg.iters)
    meth, lk = kappa_log10(x, y, a, b, lam, N, cfg, cfg.iters)
    nf = nfft_ref.sinkhorn_fastsum(x, y, a, b, lam, N, cfg.eps_B, cfg.p, cfg.iters, window=(cfg.m_w, cfg.sigma))
    rec = {"config": cfg.name, "n": int(x.shape[0]), "m": int(y.shape[0]), "lam": lam, "N": N,
           "iters": cfg.iters, "dense_s_cost": ref["s_cost"], "dense_s_dual": ref["s_dual"],
           "method_s_cost": meth["s_cost"], "method_s_dual": meth["s_dual"],
           "method_rel_err_s_cost": abs(meth["s_cost"] - ref["s_cost"]) / abs(ref["s_cost"]),
           "method_rel_err_s_dual": abs(meth["s_dual"] - ref["s_dual"]) / abs(ref["s_dual"]),
           "nfft_s_cost": nf["s_cost"], "nfft_s_dual": nf["s_dual"],
           "nfft_rel_err_s_cost": abs(nf["s_cost"] - ref["s_cost"]) / abs(ref["s_cost"]),
           "nfft_rel_err_s_dual": abs(nf["s_dual"] - ref["s_dual"]) / abs(ref["s_dual"]),
           "nfft_vs_method_s_cost": abs(nf["s_cost"] - meth["s_cost"]) / abs(ref["s_cost"]),
           "log10_kappa": lk, "seconds": time.time() - t0}
    print(name, json.dumps(rec), flush=True)
    return rec


def main():
    gold = {}
    cfg = get("c1")
    x, y, a, b = make_inputs(cfg)
    for N in (64, 96):
        gold[f"c1_N{N}"] = case(f"c1_N{N}", cfg, x, y, a, b, cfg.lam, N)
    for name in ("c2", "c4"):
        cfg = get(name)
        x, y, a, b = small_subsample(cfg, *make_inputs(cfg), K_SUB)
        for lam in LAMS[name]:
            gold[f"{name}_sub{K_SUB}_lam{lam:g}"] = case(name, cfg, x, y, a, b, lam, cfg.N)
            with open(OUT, "w") as fh:
                json.dump({"source": "tools/make_golden_method.py (oracle.dense.sinkhorn_divergence, "
                                     "oracle.nfft_ref.sinkhorn_fastsum)", "k_sub": K_SUB, "cases": gold},
                          fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
