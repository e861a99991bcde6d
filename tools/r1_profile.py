"""r = 1 (Laplace kernel + near field, NEXT-2) on d = 1 / 2 workloads shaped like the paper's
Table 1 / 2 experiments: plan time, per-stage fast-summation times and Sinkhorn it/s.

    python tools/r1_profile.py [--d 1] [--n 100000] [--iters 50]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, default=1)
    ap.add_argument("--n", type=int, default=100000)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--N", type=int, default=256)
    ap.add_argument("--lam", type=float, default=20.0)
    ap.add_argument("--near", type=int, default=16)
    args = ap.parse_args()
    from paper_2201_07524_b200 import capi
    rng = np.random.default_rng(7)
    x = rng.random((args.n, args.d))
    y = np.clip(rng.normal(0.5, 0.1, size=(args.n, args.d)), 0, 1)
    a = np.full(args.n, 1.0 / args.n)
    b = a.copy()
    ctx = capi.Context(0)
    dev = lambda z: torch.from_numpy(np.ascontiguousarray(z)).cuda()  # noqa: E731
    dx, dy, da, db = dev(x), dev(y), dev(a), dev(b)
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        P = capi.Plan(ctx, dx, dy, args.lam, args.N, 2.0, 8, 1 / 16, 8, r=1, near_cells=args.near)
        torch.cuda.synchronize()
        print(f"plan {rep}: {1e3 * (time.perf_counter() - t0):.2f} ms")
        if rep == 0:
            P.close()
    capi.sk_profile(True)
    for _ in range(5):
        capi.fastsum_apply(P, db, 0, 0)
        capi.fastsum_apply(P, da, 1, 0)
    torch.cuda.synchronize()
    for s, (c, ms) in capi.sk_profile_read().items():
        if c:
            print(f"{s:10s} launches {c:4d}  avg {ms / c:9.4f} ms")
    capi.sk_profile(False)
    u, v, info = capi.sinkhorn_run(P, da, db, 3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    u, v, info = capi.sinkhorn_run(P, da, db, args.iters)
    e1.record()
    torch.cuda.synchronize()
    print(f"sinkhorn_run r=1 d={args.d} n={args.n}: {args.iters / (e0.elapsed_time(e1) * 1e-3):.1f} it/s, "
          f"kappa {info.kappa_log10_est:.2f}")


if __name__ == "__main__":
    main()
