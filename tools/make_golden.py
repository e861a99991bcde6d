"""Write tests/golden/divergence_full.json: oracle divergences of the BASELINE.json workloads at
full size (c2, 1e5 points per side) or on the seeded 1e5-point subsample (c3, c5; BJ north_star).

Calls only oracle/ (and the synthetic input generators). Long-running (about an hour per
workload on 8 cores); run in the background:

    nice python tools/make_golden.py c2 c5
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import dense  # noqa: E402
from synthetic import get, make_inputs, subsample  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "divergence_full.json")
# relative tolerance the GPU must meet (1e-8 = BJ gate; c2 is conditioning-limited)
TOL = {"c2": 1e-5, "c3": 1e-8, "c4": 1e-3, "c5": 1e-8}
TOL_DUAL = {"c2": 1e-7, "c3": 1e-8, "c4": 1e-4, "c5": 1e-8}


def main(names):
    gold = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for name in names:
        cfg = get(name)
        x, y, a, b = make_inputs(cfg)
        sub = cfg.n > 100_000
        if sub:
            x, y, a, b = subsample(cfg, x, y, a, b)
        t0 = time.time()
        res, f, g = dense.sinkhorn_divergence(x, y, a, b, cfg.lam, cfg.iters)
        dt = time.time() - t0
        gold[name] = {
            "s_cost": res["s_cost"], "s_dual": res["s_dual"], "row_resid": res["row_resid"],
            "mass": res["mass"], "subsample": sub, "n": int(x.shape[0]), "m": int(y.shape[0]),
            "iters": cfg.iters, "tol": TOL[name], "tol_dual": TOL_DUAL[name], "enonpos_allowed": name == "c4", "oracle_seconds": dt, "oracle_threads": dense.num_threads(),
            "source": "tools/make_golden.py -> oracle.dense.sinkhorn_divergence (log-domain Alg. 1, P:L261-291)",
        }
        with open(OUT, "w") as fh:
            json.dump(gold, fh, indent=1, sort_keys=True)
        print(name, gold[name], flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c2"])
