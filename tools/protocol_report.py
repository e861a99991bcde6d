"""Parity report at BASELINE.json's protocol on one B200 (the numbers behind DESIGN.md §8):

* matvecs: 4096 seeded rows x both directions x both kernels x weights (i)/(ii) against the
  oracle goldens (tests/golden/matvec_<cfg>.npz) for c3/c4/c5, full matvecs for c1/c2, and
  weights (iii) (the GPU's converged iterate) on 1024 rows against the oracle at run time;
* divergences: s~ and s on BJ's 1e5-point subsamples (tests/golden/divergence_full.json);
* conditioning: c1 at N = 64 / 96 and the c2 / c4 lambda sweeps against the oracle's three
  statements (tests/golden/method_envelope.json), with the GPU's kappa estimates.

    python tools/protocol_report.py > profiles/r2_parity_protocol.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import dense  # noqa: E402
from synthetic import check_rows, get, make_inputs, small_subsample, subsample, uniform_test_weights  # noqa: E402
from synthetic.configs import CONFIG_INDEX  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")


def rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


def main():
    from paper_2201_07524_b200 import capi
    ctx = capi.Context(0)
    dev = lambda z: torch.from_numpy(np.ascontiguousarray(z, dtype=np.float64)).cuda()  # noqa: E731
    plan = lambda cfg, x, y, N=None: capi.Plan(ctx, dev(x), dev(y), cfg.lam, N or cfg.N, cfg.sigma,  # noqa: E731
                                               cfg.m_w, cfg.eps_B, cfg.p)
    out = {"matvec": {}, "divergence": {}, "c1": {}, "sweep": {}}
    # ---- matvecs
    for name in ("c1", "c2", "c3", "c4", "c5"):
        cfg = get(name)
        ci = CONFIG_INDEX[name]
        x, y, a, b = make_inputs(cfg)
        P = plan(cfg, x, y)
        rec = {}
        wts = {"marginal": (b, a), "uniform01": (uniform_test_weights(ci, y.shape[0]), uniform_test_weights(ci, x.shape[0], 1))}
        path = os.path.join(GOLD, f"matvec_{name}.npz")
        gold = np.load(path) if os.path.exists(path) else None
        for wname, (wy, wx) in wts.items():
            for k in (0, 1):
                t = capi.fastsum_apply(P, dev(wy), 0, k).cpu().numpy()
                tt = capi.fastsum_apply(P, dev(wx), 1, k).cpu().numpy()
                if gold is not None:
                    e = (rel(t[gold["rows_x"]], gold[f"t_{wname}_k{k}"]), rel(tt[gold["rows_y"]], gold[f"tt_{wname}_k{k}"]))
                    rows = 4096
                else:   # n, m <= 1e5: full matvecs against the direct sum
                    e = (rel(t, dense.direct_sum(x, y, wy, cfg.lam, k)), rel(tt, dense.direct_sum(y, x, wx, cfg.lam, k)))
                    rows = "all"
                rec[f"{wname}_k{k}"] = {"Kv": e[0], "KTu": e[1], "rows": rows}
        u, v, info = capi.sinkhorn_run(P, dev(a), dev(b), cfg.iters)
        u, v = u.cpu().numpy(), v.cpu().numpy()
        rx, ry = check_rows(ci, 1024, x.shape[0], seed=2), check_rows(ci, 1024, y.shape[0], seed=3)
        for k in ((0,) if name == "c5" else (0, 1)):
            t = capi.fastsum_apply(P, dev(v), 0, k).cpu().numpy()
            tt = capi.fastsum_apply(P, dev(u), 1, k).cpu().numpy()
            rec[f"converged_k{k}"] = {"Kv": rel(t[rx], dense.direct_sum(x, y, v, cfg.lam, k, rows=rx)),
                                      "KTu": rel(tt[ry], dense.direct_sum(y, x, u, cfg.lam, k, rows=ry)), "rows": 1024}
        rec["kappa_log10"] = [info.kappa_log10_est, info.kappa_u_log10_est]
        rec["band_tail"] = list(P.info()["band_tail"])
        P.close()
        out["matvec"][name] = rec
        print(name, "matvec worst", max(max(r["Kv"], r["KTu"]) for kk, r in rec.items() if isinstance(r, dict)),
              file=sys.stderr, flush=True)
    # ---- divergences on BJ's subsamples
    gold = json.load(open(os.path.join(GOLD, "divergence_full.json")))
    for name, g in sorted(gold.items()):
        cfg = get(name)
        x, y, a, b = make_inputs(cfg)
        if g.get("subsample"):
            x, y, a, b = subsample(cfg, x, y, a, b)
        P = plan(cfg, x, y)
        try:
            u, v, info = capi.sinkhorn_run(P, dev(a), dev(b), cfg.iters)
            sd, sc = capi.sinkhorn_divergence(P, dev(a), dev(b), u, v)
            out["divergence"][name] = {"n": int(x.shape[0]), "m": int(y.shape[0]), "s_cost": sc, "s_dual": sd,
                                       "s_cost_rel_err": abs(sc - g["s_cost"]) / abs(g["s_cost"]),
                                       "s_dual_rel_err": abs(sd - g["s_dual"]) / abs(g["s_dual"]),
                                       "tol": g["tol"], "tol_dual": g.get("tol_dual"),
                                       "kappa_log10": [info.kappa_log10_est, info.kappa_u_log10_est]}
        except capi.SkError as e:
            out["divergence"][name] = {"error": str(e), "bad_iter": e.info.bad_iter if e.info else None}
        P.close()
    # ---- conditioning
    meth = json.load(open(os.path.join(GOLD, "method_envelope.json")))["cases"]
    cfg = get("c1")
    x, y, a, b = make_inputs(cfg)
    for N in (64, 96):
        r = meth[f"c1_N{N}"]
        P = plan(cfg, x, y, N)
        u, v, info = capi.sinkhorn_run(P, dev(a), dev(b), cfg.iters)
        sd, sc = capi.sinkhorn_divergence(P, dev(a), dev(b), u, v)
        out["c1"][f"N{N}"] = {"gpu_vs_dense": abs(sc - r["dense_s_cost"]) / r["dense_s_cost"],
                              "gpu_vs_nfft_method": abs(sc - r["nfft_s_cost"]) / r["nfft_s_cost"],
                              "gpu_vs_ndft_method": abs(sc - r["method_s_cost"]) / r["method_s_cost"],
                              "ndft_method_vs_dense": r["method_rel_err_s_cost"], "nfft_method_vs_dense": r["nfft_rel_err_s_cost"],
                              "nfft_vs_ndft": r["nfft_vs_method_s_cost"],
                              "s_dual_gpu_vs_dense": abs(sd - r["dense_s_dual"]) / abs(r["dense_s_dual"]),
                              "kappa_log10": [info.kappa_log10_est, info.kappa_u_log10_est],
                              "band_tail": list(P.info()["band_tail"])}
        P.close()
    for name in ("c2", "c4"):
        cfg = get(name)
        x, y, a, b = small_subsample(cfg, *make_inputs(cfg), 3000)
        rows = []
        for key, r in sorted(((k, v) for k, v in meth.items() if k.startswith(f"{name}_sub")), key=lambda kv: kv[1]["lam"]):
            P = plan(cfg.with_(lam=r["lam"]), x, y)
            row = {"lam": r["lam"], "oracle_log10_kappa": r["log10_kappa"],
                   "ndft_method_vs_dense": r["method_rel_err_s_cost"], "nfft_method_vs_dense": r["nfft_rel_err_s_cost"]}
            try:
                u, v, info = capi.sinkhorn_run(P, dev(a), dev(b), cfg.iters)
                sd, sc = capi.sinkhorn_divergence(P, dev(a), dev(b), u, v)
                row.update(gpu_vs_dense=abs(sc - r["dense_s_cost"]) / r["dense_s_cost"],
                           gpu_kappa_log10=[info.kappa_log10_est, info.kappa_u_log10_est])
            except capi.SkError as e:
                row.update(gpu_error=str(e).split(":")[0], bad_iter=e.info.bad_iter if e.info else None)
            P.close()
            rows.append(row)
        out["sweep"][name] = rows
    print(json.dumps(out, indent=1, default=float))
    ctx.close()


if __name__ == "__main__":
    main()
