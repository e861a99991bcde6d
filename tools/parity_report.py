"""Parity report of the CUDA path against the CPU oracle on every BASELINE.json workload.

For each config: full-size plan; matvec rel-l_inf on seeded rows (both directions, both kernels,
b/a and U(0,1) weights); Sinkhorn divergence on an oracle-sized subsample (first k points,
renormalised weights) at the config's lambda / NFFT parameters, with the GPU's kappa estimate.
Writes a JSON report (profiles/) and prints a table.

    python tools/parity_report.py [--k 3000] [--rows 1024] [--out profiles/r1_parity.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import dense  # noqa: E402
from synthetic import check_rows, get, make_inputs, uniform_test_weights  # noqa: E402
from synthetic.configs import CONFIG_INDEX  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def rel(got, ref):
    return float(np.abs(got - ref).max() / np.abs(ref).max())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=int, default=3000)
    ap.add_argument("--rows", type=int, default=1024)
    ap.add_argument("--configs", default="c1,c2,c3,c4,c5")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r1_parity.json"))
    args = ap.parse_args()
    from paper_2201_07524_b200 import capi
    ctx = capi.Context(0)
    report = {}
    for name in args.configs.split(","):
        cfg = get(name)
        ci = CONFIG_INDEX[name]
        rec = {"config": cfg.asdict()}
        t0 = time.time()
        x, y, a, b = make_inputs(cfg)
        P = capi.Plan(ctx, dev(x), dev(y), cfg.lam, cfg.N, cfg.sigma, cfg.m_w, cfg.eps_B, cfg.p)
        rows_x = check_rows(ci, min(args.rows, x.shape[0]), x.shape[0])
        rows_y = check_rows(ci, min(args.rows, y.shape[0]), y.shape[0], seed=1)
        mv = {}
        for wname, (wy, wx) in {"marginal": (b, a),
                                "uniform01": (uniform_test_weights(ci, y.shape[0]),
                                              uniform_test_weights(ci, x.shape[0], 1))}.items():
            for kernel in (0, 1):
                t = capi.fastsum_apply(P, dev(wy), 0, kernel).cpu().numpy()
                e1 = rel(t[rows_x], dense.direct_sum(x, y, wy, cfg.lam, kernel, rows=rows_x))
                tt = capi.fastsum_apply(P, dev(wx), 1, kernel).cpu().numpy()
                e2 = rel(tt[rows_y], dense.direct_sum(y, x, wx, cfg.lam, kernel, rows=rows_y))
                mv[f"K{kernel}_{wname}"] = [e1, e2]
        rec["matvec_rel_linf"] = mv
        rec["matvec_rows"] = [int(rows_x.shape[0]), int(rows_y.shape[0])]
        P.close()
        del x, y, a, b
        # divergence on the oracle-sized subsample
        k = min(args.k, cfg.n, cfg.m)
        grid_like = cfg.x_dist in ("jitter_grid", "pixel_grid")
        xs, ys, as_, bs = make_inputs(cfg.with_(n=min(cfg.n, 4 * k), m=min(cfg.m, 4 * k))) if not grid_like else (None,) * 4
        if grid_like:
            # c4 is a jittered grid: take every (K/k')-th row and column block of the full grid
            x, y, a, b = make_inputs(cfg)
            idx = np.random.default_rng(0).choice(x.shape[0], size=k, replace=False)
            idy = np.random.default_rng(1).choice(y.shape[0], size=k, replace=False)
            xs, ys, as_, bs = x[np.sort(idx)], y[np.sort(idy)], a[np.sort(idx)], b[np.sort(idy)]
            del x, y, a, b
        xs, ys = xs[:k], ys[:k]
        as_, bs = as_[:k] / as_[:k].sum(), bs[:k] / bs[:k].sum()
        ref, _, _ = dense.sinkhorn_divergence(xs, ys, as_, bs, cfg.lam, cfg.iters)
        P = capi.Plan(ctx, dev(xs), dev(ys), cfg.lam, cfg.N, cfg.sigma, cfg.m_w, cfg.eps_B, cfg.p)
        try:
            u, v, info = capi.sinkhorn_run(P, dev(as_), dev(bs), cfg.iters)
            sd, sc = capi.sinkhorn_divergence(P, dev(as_), dev(bs), u, v)
            rec["divergence"] = {"k": k, "s_cost": sc, "s_cost_oracle": ref["s_cost"],
                                 "s_cost_rel_err": abs(sc - ref["s_cost"]) / abs(ref["s_cost"]),
                                 "s_dual": sd, "s_dual_oracle": ref["s_dual"],
                                 "s_dual_rel_err": abs(sd - ref["s_dual"]) / abs(ref["s_dual"]),
                                 "kappa_log10": info.kappa_log10_est, "status": "SK_OK"}
        except capi.SkError as e:
            rec["divergence"] = {"k": k, "status": str(e), "s_cost_oracle": ref["s_cost"],
                                 "kappa_log10": e.info.kappa_log10_est if e.info else None}
        P.close()
        rec["seconds"] = time.time() - t0
        report[name] = rec
        d = rec["divergence"]
        worst = max(max(v) for v in mv.values())
        worstK0 = max(max(v) for kk, v in mv.items() if kk.startswith("K0"))
        print(f"{name}: matvec worst K {worstK0:.2e} (all incl. c*K {worst:.2e}); divergence k={k}: "
              f"{d.get('status')} s~ rel {d.get('s_cost_rel_err', float('nan')):.2e} "
              f"s rel {d.get('s_dual_rel_err', float('nan')):.2e} log10 kappa {d.get('kappa_log10')}", flush=True)
    with open(args.out, "w") as fh:
        json.dump(report, fh, indent=1)
    ctx.close()


if __name__ == "__main__":
    main()
