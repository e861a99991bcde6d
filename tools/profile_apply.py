"""Small driver for ncu / timing: plan one workload and run a few fast-summation applies.

    python tools/profile_apply.py --config c3 --reps 3 [--n 1000000 --m 1000000]
Prints per-stage CUDA-event times from the library profiler.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from synthetic import get, make_inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--m", type=int, default=0)
    ap.add_argument("--per-dir", action="store_true", help="also time K v and K^T u separately")
    args = ap.parse_args()
    from paper_2201_07524_b200 import capi
    cfg = get(args.config)
    if args.n:
        cfg = cfg.with_(n=args.n, m=args.m or args.n)
    x, y, a, b = make_inputs(cfg)
    ctx = capi.Context(0)
    t = lambda z: torch.from_numpy(np.ascontiguousarray(z)).cuda()  # noqa: E731
    import time
    dx, dy = t(x), t(y)
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        P = capi.Plan(ctx, dx, dy, cfg.lam, cfg.N, cfg.sigma, cfg.m_w, cfg.eps_B, cfg.p)
        torch.cuda.synchronize()
        print(f"plan {rep}: {1e3 * (time.perf_counter() - t0):.1f} ms")
        if rep == 0:
            P.close()
    w_y, w_x = t(b), t(a)
    capi.fastsum_apply(P, w_y, 0, 0)
    torch.cuda.synchronize()
    capi.sk_profile(True)
    for _ in range(args.reps):
        capi.fastsum_apply(P, w_y, 0, 0)
        capi.fastsum_apply(P, w_x, 1, 0)
    torch.cuda.synchronize()
    prof = capi.sk_profile_read()
    for s, (c, ms) in prof.items():
        if c:
            print(f"{s:10s} launches {c:4d}  avg {ms / c:9.4f} ms")
    if args.per_dir:   # spread y + interp x (K v), then spread x + interp y (K^T u)
        for tr, w_ in ((0, w_y), (1, w_x)):
            for _ in range(args.reps):
                capi.fastsum_apply(P, w_, tr, 0)
            torch.cuda.synchronize()
            prof = capi.sk_profile_read()
            print(f"  dir {tr}: " + "  ".join(f"{s} {ms / c:.4f}" for s, (c, ms) in prof.items() if c and s in ("spread", "interp")))
    P.close()
    ctx.close()


if __name__ == "__main__":
    main()
