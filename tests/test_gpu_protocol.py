"""GPU parity at BASELINE.json's protocol (north_star; SURVEY.md §8(d) "Parity protocol"), and
the evidence that the divergence misses on c1 (N = 64), c2 and c4 are the method's.

* Matvecs above 1e5 points: 4096 seeded target rows against the direct sum over all sources,
  both directions, both kernels, weights (i) b / a and (ii) U(0,1) from oracle-only goldens
  (tools/make_golden_matvec.py -> tests/golden/matvec_<cfg>.npz); weights (iii), the GPU's own
  converged iterate, on >= 1024 fresh seeded rows with the oracle evaluated at test time.
  Gate: relative l_inf <= 1e-9.
* Divergences against the oracle on BJ's seeded 1e5-point subsamples (golden/divergence_full.json):
  s~ and s both asserted.
* Conditioning (SURVEY §8(c) consequence (1)): oracle.nfft_ref.sinkhorn_fastsum runs Alg. 2 on
  the method's own fast summation (exact NDFTs, and the full NFFT with its window). On c1 at
  N = 64 the GPU lies within the spread of those two statements while all of them miss the
  dense oracle by 6e-5: the Fourier truncation. On the c2 / c4 subsamples a lambda sweep shows
  the error tracking kappa: within 1e-8 wherever log10 kappa <= 8, and within a small multiple
  of the method's own spread elsewhere (golden/method_envelope.json, tools/make_golden_method.py).
"""
import json
import os

import numpy as np
import pytest
import torch

from oracle import dense
from synthetic import check_rows, get, make_inputs, small_subsample, subsample, uniform_test_weights
from synthetic.configs import CONFIG_INDEX

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
MATVEC_TOL = 1e-9


@pytest.fixture(scope="module")
def capi(cuda_ok):
    from paper_2201_07524_b200 import capi as C
    return C


@pytest.fixture(scope="module")
def ctx(capi):
    c = capi.Context(0)
    yield c
    c.close()


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def rel_linf(got, ref):
    return float(np.abs(got - ref).max() / np.abs(ref).max())


def _plan(capi, ctx, cfg, x, y, N=None):
    return capi.Plan(ctx, dev(x), dev(y), cfg.lam, N or cfg.N, cfg.sigma, cfg.m_w, cfg.eps_B, cfg.p)


# ------------------------------------------------------------------ matvecs: 4096-row goldens + (iii)
def _matvec_protocol(capi, ctx, name, rows_iii, kernels_iii=(0, 1), rows_iii_k1=None):
    path = os.path.join(GOLDEN, f"matvec_{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated (tools/make_golden_matvec.py)")
    gold = np.load(path)
    meta = json.loads(str(gold["meta"]))
    cfg = get(name)
    ci = CONFIG_INDEX[name]
    x, y, a, b = make_inputs(cfg)
    assert meta["n"] == x.shape[0] and meta["m"] == y.shape[0]
    rx, ry = gold["rows_x"], gold["rows_y"]
    assert np.array_equal(rx, check_rows(ci, 4096, x.shape[0])) and np.array_equal(ry, check_rows(ci, 4096, y.shape[0], seed=1))
    P = _plan(capi, ctx, cfg, x, y)
    errs = {}
    weights = {"marginal": (b, a),
               "uniform01": (uniform_test_weights(ci, y.shape[0]), uniform_test_weights(ci, x.shape[0], 1))}
    for wname, (wy, wx) in weights.items():
        for kernel in (0, 1):
            t = capi.fastsum_apply(P, dev(wy), 0, kernel).cpu().numpy()
            tt = capi.fastsum_apply(P, dev(wx), 1, kernel).cpu().numpy()
            errs[(wname, kernel)] = (rel_linf(t[rx], gold[f"t_{wname}_k{kernel}"]),
                                     rel_linf(tt[ry], gold[f"tt_{wname}_k{kernel}"]))
    # (iii) the GPU's own converged iterate: u, v after the config's iteration count
    u, v, info = capi.sinkhorn_run(P, dev(a), dev(b), cfg.iters)
    u, v = u.cpu().numpy(), v.cpu().numpy()
    r3x = check_rows(ci, rows_iii, x.shape[0], seed=2)
    r3y = check_rows(ci, rows_iii, y.shape[0], seed=3)
    for kernel in kernels_iii:
        if kernel == 1 and rows_iii_k1:
            r3x, r3y = r3x[:: max(1, len(r3x) // rows_iii_k1)], r3y[:: max(1, len(r3y) // rows_iii_k1)]
        t = capi.fastsum_apply(P, dev(v), 0, kernel).cpu().numpy()
        tt = capi.fastsum_apply(P, dev(u), 1, kernel).cpu().numpy()
        errs[("converged", kernel)] = (rel_linf(t[r3x], dense.direct_sum(x, y, v, cfg.lam, kernel, rows=r3x)),
                                       rel_linf(tt[r3y], dense.direct_sum(y, x, u, cfg.lam, kernel, rows=r3y)))
    P.close()
    bad = {k: e for k, e in errs.items() if max(e) > MATVEC_TOL}
    assert not bad, (name, errs, info.asdict())
    return errs


def test_matvec_protocol_c3(capi, ctx):
    _matvec_protocol(capi, ctx, "c3", 1024)


def test_matvec_protocol_c4(capi, ctx):
    _matvec_protocol(capi, ctx, "c4", 1024)


def test_matvec_protocol_c5(capi, ctx):
    """c5 at full size (1e8 + 8e7 nodes, the bench's plan). Weights (iii) on 1024 rows per
    direction for kernel 0 (the Sinkhorn kernel) and 256 rows for c exp(-lam c): the oracle
    evaluates them at test time (1024 x 1.8e8 pair sums per kernel)."""
    _matvec_protocol(capi, ctx, "c5", 1024, rows_iii_k1=256)


def test_matvec_converged_weights_c2(capi, ctx):
    """c2 (1e5 points: full matvecs against the direct sum) with weights (iii) on 1024 rows; (i)
    and (ii) on all rows are test_gpu_parity.test_matvec_parity_full_size."""
    cfg = get("c2")
    ci = CONFIG_INDEX["c2"]
    x, y, a, b = make_inputs(cfg)
    P = _plan(capi, ctx, cfg, x, y)
    u, v, info = capi.sinkhorn_run(P, dev(a), dev(b), cfg.iters)
    u, v = u.cpu().numpy(), v.cpu().numpy()
    rx, ry = check_rows(ci, 1024, x.shape[0], seed=2), check_rows(ci, 1024, y.shape[0], seed=3)
    for kernel in (0, 1):
        t = capi.fastsum_apply(P, dev(v), 0, kernel).cpu().numpy()
        tt = capi.fastsum_apply(P, dev(u), 1, kernel).cpu().numpy()
        e = (rel_linf(t[rx], dense.direct_sum(x, y, v, cfg.lam, kernel, rows=rx)),
             rel_linf(tt[ry], dense.direct_sum(y, x, u, cfg.lam, kernel, rows=ry)))
        assert max(e) <= MATVEC_TOL, (kernel, e, info.asdict())


# ------------------------------------------------------------------ divergences on BJ's subsamples
def test_divergence_golden_full_both_values(capi, ctx):
    """s~ and s on BJ's seeded 1e5-point subsamples (c3, c4, c5) and full c2 against the
    oracle's log-domain Alg. 1 (golden/divergence_full.json, tools/make_golden.py). Gates: 1e-8
    where Alg. 2 is conditioned (c3, c5); the method envelope on c2 / c4, whose size the
    conditioning tests below establish from the oracle alone."""
    gold = json.load(open(os.path.join(GOLDEN, "divergence_full.json")))
    for name, rec in sorted(gold.items()):
        cfg = get(name)
        x, y, a, b = make_inputs(cfg)
        if rec.get("subsample"):
            x, y, a, b = subsample(cfg, x, y, a, b)
        P = _plan(capi, ctx, cfg, x, y)
        da, db = dev(a), dev(b)
        try:
            u, v, info = capi.sinkhorn_run(P, da, db, cfg.iters)
        except capi.SkError as e:   # c4: Alg. 2 may break down in FP64
            assert e.code == capi.SK_ENONPOS and rec.get("enonpos_allowed"), (name, str(e))
            P.close()
            continue
        sd, sc = capi.sinkhorn_divergence(P, da, db, u, v)
        P.close()
        e_c = abs(sc - rec["s_cost"]) / abs(rec["s_cost"])
        e_d = abs(sd - rec["s_dual"]) / abs(rec["s_dual"])
        assert e_c <= rec["tol"], (name, "s_cost", sc, rec, info.asdict())
        assert e_d <= rec["tol_dual"], (name, "s_dual", sd, rec, info.asdict())


# ------------------------------------------------------------------ conditioning: the method's own error
def _method_golden():
    path = os.path.join(GOLDEN, "method_envelope.json")
    if not os.path.exists(path):
        pytest.skip("golden/method_envelope.json not generated (tools/make_golden_method.py)")
    return json.load(open(path))["cases"]


@pytest.mark.parametrize("N", [64, 96])
def test_c1_equals_method_statement(capi, ctx, N):
    """c1 (d = 1, lam = 100, kappa ~ 10^7.8) at BJ's N = 64 and at N = 96, against three oracle
    statements on the same inputs (golden/method_envelope.json): dense Alg. 1, Alg. 2 on the
    method's fast summation with exact NDFTs (`method`) and with the full NFFT incl. the window
    (`nfft`). `method` and `nfft` differ only by the window error (~5e-15 per matvec), yet their
    s~ differ by ~1e-8 at N = 64 (4e-10 at N = 96): at this kappa FP64-level matvec perturbations
    move s~ that much. The GPU's matvec differs from `nfft` by the same ~5e-15 (FP64 rounding), so
    it must lie within 5 x that spread + 1e-9 of `nfft`, and at N = 64 its
    distance to dense must be the method's Fourier truncation: within 0.1 % of `method`'s
    (6.4e-5 in s~; exp(-pi^2 32^2 / lam') of c exp(-lam c), reading Q9). At N = 96
    the truncation is gone and the GPU meets 1e-8 against dense."""
    rec = _method_golden()[f"c1_N{N}"]
    cfg = get("c1")
    x, y, a, b = make_inputs(cfg)
    P = _plan(capi, ctx, cfg, x, y, N=N)
    da, db = dev(a), dev(b)
    u, v, info = capi.sinkhorn_run(P, da, db, cfg.iters)
    sd, sc = capi.sinkhorn_divergence(P, da, db, u, v)
    spread_c = abs(rec["nfft_s_cost"] - rec["method_s_cost"]) / abs(rec["nfft_s_cost"])
    spread_d = abs(rec["nfft_s_dual"] - rec["method_s_dual"]) / abs(rec["nfft_s_dual"])
    e_nf_c = abs(sc - rec["nfft_s_cost"]) / abs(rec["nfft_s_cost"])
    e_nf_d = abs(sd - rec["nfft_s_dual"]) / abs(rec["nfft_s_dual"])
    print(f"c1 N={N}: gpu-nfft s~ {e_nf_c:.2e} (spread {spread_c:.2e}) s {e_nf_d:.2e} (spread {spread_d:.2e})")
    assert e_nf_c <= 5 * spread_c + 1e-9, (sc, rec)
    assert e_nf_d <= 5 * spread_d + 1e-9, (sd, rec)
    e_c = abs(sc - rec["dense_s_cost"]) / abs(rec["dense_s_cost"])
    e_d = abs(sd - rec["dense_s_dual"]) / abs(rec["dense_s_dual"])
    if N == 64:   # the method's own miss, reproduced
        assert rec["method_rel_err_s_cost"] > 1e-5 and abs(e_c / rec["method_rel_err_s_cost"] - 1) < 1e-3, (e_c, rec)
    else:
        assert e_c <= 1e-8 and e_d <= 1e-8, (e_c, e_d, rec)
    # the plan's accuracy report flags N = 64: the c exp(-lam c) band tail is ~1e-9 absolute
    tail = P.info()["band_tail"]
    assert (tail[1] > 1e-10) if N == 64 else (tail[1] < 1e-13), tail


@pytest.mark.parametrize("name", ["c2", "c4"])
def test_conditioning_lambda_sweep(capi, ctx, name):
    """c2 / c4 on their seeded 3000-point subsamples at lam in {5, 10, 20, 50, 100, 200} (their
    BJ lambda included) and the config's NFFT parameters. Per lambda, the GPU's relative s~
    error against the dense oracle is
      <= 1e-8 wherever log10 kappa <= 8 (the BJ gate holds wherever Alg. 2 is conditioned), and
      <= 10 x the method's own spread + 1e-10 everywhere, the spread being the largest distance
         among the oracle's three statements (dense, `method` = exact-NDFT fast summation, `nfft`
         = full NFFT fast summation): the GPU stays inside the method's envelope,
    with kappa from the oracle's run (golden/method_envelope.json). A breakdown (SK_ENONPOS) is
    accepted only where log10 kappa > 12; where the oracle's own Alg. 2 on the method's fast
    summation breaks down (a non-positive denominator: kappa = inf) any GPU
    outcome is the method's."""
    cases = {k: v for k, v in _method_golden().items() if k.startswith(f"{name}_sub")}
    assert len(cases) >= 6
    cfg = get(name)
    x, y, a, b = small_subsample(cfg, *make_inputs(cfg), 3000)
    rows = []
    for key, rec in sorted(cases.items(), key=lambda kv: kv[1]["lam"]):
        assert rec["n"] == x.shape[0] and rec["m"] == y.shape[0]
        P = _plan(capi, ctx, cfg.with_(lam=rec["lam"]), x, y)
        da, db = dev(a), dev(b)
        spread = float(np.nanmax([rec["method_rel_err_s_cost"], rec["nfft_rel_err_s_cost"], rec["nfft_vs_method_s_cost"]]))
        broken = not np.isfinite(rec["log10_kappa"])
        try:
            u, v, info = capi.sinkhorn_run(P, da, db, cfg.iters)
        except capi.SkError as e:
            assert e.code == capi.SK_ENONPOS and rec["log10_kappa"] > 12, (key, str(e))
            rows.append((rec["lam"], round(rec["log10_kappa"], 2), None, spread))
            P.close()
            continue
        sd, sc = capi.sinkhorn_divergence(P, da, db, u, v)
        P.close()
        err = abs(sc - rec["dense_s_cost"]) / abs(rec["dense_s_cost"])
        rows.append((rec["lam"], round(rec["log10_kappa"], 2), err, spread))
        if broken:
            continue
        if rec["log10_kappa"] <= 8:
            assert err <= 1e-8, (key, err, rec)
        assert err <= 10 * spread + 1e-10, (key, err, spread, rec)
    print(name, "(lam, log10 kappa, gpu s~ err, method spread):", rows)
    assert any(r[1] <= 8 for r in rows) and any(r[1] > 8 for r in rows), rows   # both regimes covered
