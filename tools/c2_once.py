"""One c2 solve (plan + 5 iterations + divergence) for ncu launch lists of the small-workload path."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from synthetic import get, make_inputs  # noqa: E402

from paper_2201_07524_b200 import capi  # noqa: E402

cfg = get(sys.argv[1] if len(sys.argv) > 1 else "c2")
x, y, a, b = make_inputs(cfg)
ctx = capi.Context(0)
dev = lambda z: torch.from_numpy(np.ascontiguousarray(z)).cuda()  # noqa: E731
dx, dy, da, db = dev(x), dev(y), dev(a), dev(b)
for _ in range(2):
    r = capi.sinkhorn_solve(ctx, dx, dy, da, db, cfg.lam, cfg.N, cfg.sigma, cfg.m_w, cfg.eps_B, cfg.p, 5)
torch.cuda.synchronize()
print(r[:2])
