"""Small end-to-end runs of every kernel family for compute-sanitizer:
memcheck / racecheck / synccheck over the TMA + mbarrier spreads, the DMMA interps, the d = 1 / 2
paths, the pruned FFT, r = 1 and the Sinkhorn loop (graph replay included).

    compute-sanitizer --tool memcheck python tools/sanitize_run.py

Sizes are c1/c2-like so the instrumented run finishes in minutes. Prints one line per case and
'SANITIZE_RUN_OK' at the end.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from synthetic import get, make_inputs  # noqa: E402


def main():
    from paper_2201_07524_b200 import capi
    dev = lambda z: torch.from_numpy(np.ascontiguousarray(z, dtype=np.float64)).cuda()  # noqa: E731
    ctx = capi.Context(0)
    cases = [
        ("c1 d=1", get("c1"), 1000, 1000, {}),
        ("c2 d=2 dmma", get("c2"), 20000, 15000, {}),
        ("c3 d=3 tmapad sparse+xpairs", get("c3"), 20000, 20000, {}),
        ("c5 d=3 tmapad dense", get("c5"), 60000, 50000, {"SK_SEG_DENSE_MIN": "0"}),
        ("c5 d=3 pruned fft", get("c5"), 200000, 160000, {}),
    ]
    for name, cfg, n, m, env in cases:
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        try:
            x, y, a, b = make_inputs(cfg.with_(n=n, m=m) if cfg.n > n else cfg)
            a, b = a / a.sum(), b / b.sum()
            P = capi.Plan(ctx, dev(x), dev(y), cfg.lam, cfg.N, cfg.sigma, cfg.m_w, cfg.eps_B, cfg.p)
            t = capi.fastsum_apply(P, dev(b), 0, 1)
            g = capi.nfft_spread(P, 1, dev(b))
            ti = capi.nfft_interp(P, 0, g)
            u, v, info = capi.sinkhorn_run(P, dev(a), dev(b), 4)       # graph replay of 3 iterations
            sd, sc = capi.sinkhorn_divergence(P, dev(a), dev(b), u, v)
            torch.cuda.synchronize()
            print(f"{name}: s~ {sc:.6g} s {sd:.6g} t[0] {float(t[0]):.4g} interp[0] {float(ti[0]):.4g}", flush=True)
            P.close()
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
    # r = 1 (near field)
    rng = np.random.default_rng(0)
    x, y = rng.random((300, 2)), rng.random((280, 2))
    P = capi.Plan(ctx, dev(x), dev(y), 20.0, 64, 2.0, 8, 1 / 16, 8, r=1, near_cells=16)
    t = capi.fastsum_apply(P, dev(rng.random(280)), 0, 0)
    torch.cuda.synchronize()
    print(f"r=1 d=2: t[0] {float(t[0]):.4g}")
    P.close()
    ctx.close()
    print("SANITIZE_RUN_OK")


if __name__ == "__main__":
    main()
