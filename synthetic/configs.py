"""Config registry for the five BASELINE.json workloads (c1..c5).

Pure data: problem sizes and the NFFT / Sinkhorn parameters named in
BASELINE.json ``configs`` (readings where it is silent: SURVEY.md §8(d),
DESIGN.md "Input recipe"). No arithmetic of the method lives here; this module
is shared by the oracle side and the CUDA side only as a source of parameters.
"""
from __future__ import annotations

from dataclasses import dataclass, replace, asdict


@dataclass(frozen=True)
class Config:
    name: str
    d: int            # dimension of the support points
    n: int            # number of source-measure atoms x_i (weights a)
    m: int            # number of target-measure atoms y_j (weights b)
    lam: float        # entropic regularisation lambda (cost = squared Euclidean)
    N: int            # NFFT bandwidth per axis (even)
    sigma: float      # oversampling factor, oversampled grid = sigma*N per axis
    m_w: int          # Kaiser-Bessel window cutoff (2*m_w taps per axis)
    eps_B: float      # boundary-regularisation width (torus units)
    p: int            # two-point Taylor order of the boundary regularisation K_B
    iters: int        # Sinkhorn iterations (1 iteration = u-update + v-update)
    x_dist: str
    y_dist: str
    w_dist: str       # weight recipe ("uniform" | "dirichlet" | "bumps")
    gmm_k: int = 0    # GMM components (x side) when x_dist == "gmm"
    gmm_sigma: float = 0.0
    grid_x: int = 0   # jittered-grid side length (c4)
    grid_y: int = 0
    sub_n: int = 0    # divergence-parity subsample sizes (0 = full size)
    sub_m: int = 0
    r: int = 2            # cost |x - y|^r (NEXT-2: r = 1, Laplace kernel + near field)
    near_cells: int = 0   # r = 1: near-field radius in oversampled-grid cells

    def with_(self, **kw) -> "Config":
        return replace(self, **kw)

    def asdict(self):
        return asdict(self)


CONFIGS = {
    # BJ configs[0]: d=1, n=m=1000, lambda=100, N=64, sigma=2, m_w=8, eps_B=1/16, 200 iters
    "c1": Config("c1", 1, 1000, 1000, 100.0, 64, 2.0, 8, 1 / 16, 8, 200,
                 "uniform", "normal_clip", "uniform"),
    # BJ configs[1]: d=2, n=m=1e5, lambda=50, N=128, m_w=8, 100 iters
    "c2": Config("c2", 2, 100_000, 100_000, 50.0, 128, 2.0, 8, 1 / 16, 8, 100,
                 "gmm", "uniform", "dirichlet", gmm_k=5, gmm_sigma=0.05),
    # BJ configs[2]: d=3, n=m=1e6, lambda=20, N=64, m_w=6, 100 iters
    "c3": Config("c3", 3, 1_000_000, 1_000_000, 20.0, 64, 2.0, 6, 1 / 16, 8, 100,
                 "normal_clip", "shell", "uniform", sub_n=100_000, sub_m=100_000),
    # BJ configs[3]: d=2, n=4e6 (2000^2), m=1732^2, lambda=200, N=256, m_w=8, 100 iters
    "c4": Config("c4", 2, 2000 * 2000, 1732 * 1732, 200.0, 256, 2.0, 8, 1 / 16, 8, 100,
                 "jitter_grid", "jitter_grid", "bumps", grid_x=2000, grid_y=1732,
                 sub_n=100_000, sub_m=75_000),
    # BJ configs[4]: d=3, n=1e8, m=8e7, lambda=30, N=128, m_w=6, 50 iters + divergence
    "c5": Config("c5", 3, 100_000_000, 80_000_000, 30.0, 128, 2.0, 6, 1 / 16, 8, 50,
                 "gmm", "uniform", "dirichlet", gmm_k=10, gmm_sigma=0.04,
                 sub_n=100_000, sub_m=80_000),
}

# the paper's image experiments (Tables 3, 6, 7) at its own
# lambda = 20, r = 2: two K x K grayscale images on the same pixel grid, pixel centres
# ((i + 1/2)/K, (j + 1/2)/K), weights = normalised gray levels. DOTmark is not in the container;
# each image is a seeded smooth bump field (the c4 recipe) standing in for it. NFFT parameters
# are the build's choice (the paper gives none): N = 64 puts the Fourier truncation of the
# Gaussian at exp(-pi^2 32^2 / lambda') ~ e^-48, m_w = 8 (FP64 window error), sigma = 2.
for _K in (32, 64, 128, 256, 512):
    CONFIGS[f"img{_K}"] = Config(f"img{_K}", 2, _K * _K, _K * _K, 20.0, 64, 2.0, 8, 1 / 16, 8, 100,
                                 "pixel_grid", "pixel_grid", "bumps", grid_x=_K, grid_y=_K)

# r = 1 on the paper's d = 1 experiment shape (Table 1, "the results for
# r = 1 are similar"): x ~ U[0,1], y ~ N(0.5, 0.1^2) clipped (the c1 recipe), uniform weights,
# lambda = 20, N = 256, m_w = 8, 16 near-field cells (DESIGN.md §9b readings R1-R6), 50 iterations.
CONFIGS["c1r1"] = Config("c1r1", 1, 100_000, 100_000, 20.0, 256, 2.0, 8, 1 / 16, 8, 50,
                         "uniform", "normal_clip", "uniform", r=1, near_cells=16)

CONFIG_INDEX = {"c1": 1, "c2": 2, "c3": 3, "c4": 4, "c5": 5,
                "img32": 6, "img64": 7, "img128": 8, "img256": 9, "img512": 10, "c1r1": 11}


def get(name: str) -> Config:
    return CONFIGS[name]
