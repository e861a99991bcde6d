"""Diagnostic: c1 at N = 64 -- GPU fast summation against the oracle's NFFT / NDFT statements of
the method and the direct sum, per matvec and along the Sinkhorn trajectory."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import dense, nfft_ref as R  # noqa: E402
from synthetic import get, make_inputs  # noqa: E402


def rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


def main():
    from paper_2201_07524_b200 import capi
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    cfg = get("c1")
    x, y, a, b = make_inputs(cfg)
    ctx = capi.Context(0)
    dev = lambda z: torch.from_numpy(np.ascontiguousarray(z)).cuda()  # noqa: E731
    P = capi.Plan(ctx, dev(x), dev(y), cfg.lam, N, cfg.sigma, cfg.m_w, cfg.eps_B, cfg.p)
    opn = R.NfftFastsumOperator(x, y, cfg.lam, N, cfg.eps_B, cfg.p, cfg.m_w, cfg.sigma)
    opd = R.FastsumOperator(x, y, cfg.lam, N, cfg.eps_B, cfg.p)
    rng = np.random.default_rng(0)
    for wname, w in (("ones", np.ones(1000)), ("rand", rng.random(1000)), ("b", b)):
        for k in (0, 1):
            g = capi.fastsum_apply(P, dev(w), 0, k).cpu().numpy()
            nf, nd = opn.apply(w, False, k), opd.apply(w, False, k)
            dr = dense.direct_sum(x, y, w, cfg.lam, k)
            print(f"{wname} k{k}: gpu-nfft {rel(g, nf):.2e} gpu-ndft {rel(g, nd):.2e} nfft-ndft {rel(nf, nd):.2e} "
                  f"gpu-direct {rel(g, dr):.2e} nfft-direct {rel(nf, dr):.2e}")
    for it in (1, 2, 5, 20, 50, 100, 200):
        u, v, info = capi.sinkhorn_run(P, dev(a), dev(b), it)
        sd, sc = capi.sinkhorn_divergence(P, dev(a), dev(b), u, v)
        rn = R.sinkhorn_fastsum(x, y, a, b, cfg.lam, N, cfg.eps_B, cfg.p, it, window=(cfg.m_w, cfg.sigma))
        rd = R.sinkhorn_fastsum(x, y, a, b, cfg.lam, N, cfg.eps_B, cfg.p, it)
        uu, vv = u.cpu().numpy(), v.cpu().numpy()
        print(f"it {it}: s~ gpu-nfft {abs(sc - rn['s_cost']) / sc:.2e} nfft-ndft {abs(rn['s_cost'] - rd['s_cost']) / sc:.2e} "
              f"| u rel {np.abs(uu / rn['alpha'] - 1).max():.2e} v rel {np.abs(vv / rn['alpha_t'] - 1).max():.2e} "
              f"| u nfft-ndft {np.abs(rn['alpha'] / rd['alpha'] - 1).max():.2e} kappa {info.kappa_log10_est:.2f}")


if __name__ == "__main__":
    main()
