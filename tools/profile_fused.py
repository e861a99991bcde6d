"""Stage times of the Sinkhorn iteration (u/v update fused into the interpolation) next to the
plain fast-summation apply, same plan, same process (stage profiler on, so no graph replay).

    python tools/profile_fused.py --config c5 --iters 4
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
    ap.add_argument("--config", default="c5")
    ap.add_argument("--iters", type=int, default=4)
    args = ap.parse_args()
    from paper_2201_07524_b200 import capi
    cfg = get(args.config)
    x, y, a, b = make_inputs(cfg)
    ctx = capi.Context(0)
    t = lambda z: torch.from_numpy(np.ascontiguousarray(z)).cuda()  # noqa: E731
    P = capi.Plan(ctx, t(x), t(y), cfg.lam, cfg.N, cfg.sigma, cfg.m_w, cfg.eps_B, cfg.p)
    da, db = t(a), t(b)
    u, v, _ = capi.sinkhorn_run(P, da, db, 2)
    torch.cuda.synchronize()
    for name, fn in (("apply (plain)", lambda: (capi.fastsum_apply(P, v, 0, 0), capi.fastsum_apply(P, u, 1, 0))),
                     ("sinkhorn_run (fused update)", lambda: capi.sinkhorn_run(P, da, db, args.iters, u=u, v=v))):
        capi.sk_profile(True)
        for _ in range(1 if "sinkhorn" in name else args.iters):
            fn()
        torch.cuda.synchronize()
        prof = capi.sk_profile_read()
        capi.sk_profile(False)
        print("==", name)
        for s, (c, ms) in prof.items():
            if c:
                print(f"   {s:10s} launches {c:4d}  avg {ms / c:9.4f} ms")
    P.close()
    ctx.close()


if __name__ == "__main__":
    main()
