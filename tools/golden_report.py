"""Divergences of the CUDA path on BJ's seeded 1e5-point subsamples (c3, c5) / full c2 against
tests/golden/divergence_full.json (written by tools/make_golden.py from the CPU oracle).

    python tools/golden_report.py > profiles/r1_golden_divergence.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from synthetic import get, make_inputs, subsample  # noqa: E402


def main():
    from paper_2201_07524_b200 import capi
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "divergence_full.json")))
    ctx = capi.Context(0)
    dev = lambda z: torch.from_numpy(np.ascontiguousarray(z)).cuda()  # noqa: E731
    out = {}
    for name, rec in gold.items():
        cfg = get(name)
        x, y, a, b = make_inputs(cfg)
        if rec.get("subsample"):
            x, y, a, b = subsample(cfg, x, y, a, b)
        P = capi.Plan(ctx, dev(x), dev(y), cfg.lam, cfg.N, cfg.sigma, cfg.m_w, cfg.eps_B, cfg.p)
        u, v, info = capi.sinkhorn_run(P, dev(a), dev(b), cfg.iters)
        sd, sc = capi.sinkhorn_divergence(P, dev(a), dev(b), u, v)
        out[name] = {"n": int(x.shape[0]), "m": int(y.shape[0]), "iters": cfg.iters,
                     "s_cost_gpu": sc, "s_cost_oracle": rec["s_cost"],
                     "s_cost_rel_err": abs(sc - rec["s_cost"]) / abs(rec["s_cost"]),
                     "s_dual_gpu": sd, "s_dual_oracle": rec["s_dual"],
                     "s_dual_rel_err": abs(sd - rec["s_dual"]) / abs(rec["s_dual"]),
                     "kappa_log10": info.kappa_log10_est, "tol": rec["tol"]}
        P.close()
    print(json.dumps(out, indent=1))
    ctx.close()


if __name__ == "__main__":
    main()
