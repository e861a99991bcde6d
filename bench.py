#!/usr/bin/env python
"""Benchmark of the NFFT fast-summation Sinkhorn hot path (arXiv 2201.07524, Alg. 2).

One STEP = one whole pass of the hot path over the workload:
plan (geometry, binning, kernel coefficients), `iters` Sinkhorn iterations (2 fast
summations each) and the divergence evaluation (2 more fast summations), via the C-ABI
entry point ``sinkhorn_solve`` on inputs already resident in HBM. ``value`` = Sinkhorn
iterations/s of the whole job (all ranks) = steps * iters / max-over-ranks device time.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]

Multi-GPU: launched by torch.distributed.run, one rank per GPU, NCCL; points are sharded by
contiguous index range and every fast summation all-reduces the oversampled grid
(strong scaling: the workload is fixed). --impl reference times the CPU oracle (dense
log-domain Alg. 1) on a bounded subsample of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from synthetic import get, make_inputs, shard_range  # noqa: E402

DEFAULT_CONFIG = os.environ.get("SK_BENCH_CONFIG", "c5")
ORACLE_PAIRS_PER_S = None   # set by cpu_oracle_rate
SMI_MS = int(os.environ.get("SK_BENCH_SMI_MS", "200"))          # clock sampling period
STAGE_PROFILE = os.environ.get("SK_BENCH_STAGE_PROFILE", "1") != "0"
FP64_FMA_PER_CLK_PER_SM = 64      # B200 FP64 vector rate
N_SM = 148
MIX_CEILING = {"spread": 31.4, "interp": 31.2}   # TF/s, DESIGN.md §6


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=None,
                   help="timed steps (default: 3 for c5; small workloads run enough steps for ~1.5 s)")
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default=DEFAULT_CONFIG)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=15.0, help="budget of the cpu_baseline sample")
    p.add_argument("--nccl-self", action="store_true",
                   help="N=1 through a one-rank NCCL communicator: the box exchange and scalar sums "
                        "run through ncclAllReduce as on N>1 (checks and times the multi-GPU path)")
    return p.parse_args()


def workload_config(cfg):
    """The `config` keys both arms report for a workload."""
    out = {"workload": cfg.name, "n": cfg.n, "m": cfg.m, "d": cfg.d, "lambda": cfg.lam, "N": cfg.N,
           "sigma": cfg.sigma, "m_w": cfg.m_w, "eps_B": cfg.eps_B, "iters_per_step": cfg.iters,
           "step": "plan + iters x (K v, K^T u) + divergence (2 applies)"}
    if cfg.r != 2:   # cost |x - y|^r: r = 1 is the Laplace kernel with its near field
        out.update({"r": cfg.r, "near_cells": cfg.near_cells})
    return out


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "fallback": True}


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None
        self.th = None

    def start(self):
        if SMI_MS <= 0:
            return
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", str(SMI_MS)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [s.strip() for s in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.th is not None:
            self.th.join(timeout=2)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[4 + k].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------- CPU oracle
def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_oracle_rate(cfg, budget_s: float):
    """Time the oracle (dense log-domain Alg. 1, as it stands) on a bounded seeded subsample
    of the workload; return (it/s extrapolated to the full workload, description)."""
    from oracle import dense
    if cfg.x_dist in ("jitter_grid", "pixel_grid"):   # grid generators need the full K x K grid
        x, y, a, b = make_inputs(cfg)
        rng = np.random.default_rng(0)
        ix = rng.permutation(x.shape[0])[:200_000]
        iy = rng.permutation(y.shape[0])[:200_000]
        x, y, a, b = x[ix], y[iy], a[ix], b[iy]
    else:
        x, y, a, b = make_inputs(cfg.with_(n=min(cfg.n, 200_000), m=min(cfg.m, 200_000)))
    # calibrate: one iteration on a small subsample, then size the sample to the budget
    k = min(2000, x.shape[0], y.shape[0])
    t0 = time.perf_counter()
    dense.sinkhorn_log(x[:k], y[:k], a[:k] / a[:k].sum(), b[:k] / b[:k].sum(), cfg.lam, 1, r=cfg.r)
    per_pair = (time.perf_counter() - t0) / (k * k)
    iters = 5
    ks = int(min(x.shape[0], y.shape[0], (budget_s / (iters * per_pair)) ** 0.5))
    ks = max(ks, 100)
    xs, ys = x[:ks], y[:ks]
    as_, bs = a[:ks] / a[:ks].sum(), b[:ks] / b[:ks].sum()
    t0 = time.perf_counter()
    dense.sinkhorn_log(xs, ys, as_, bs, cfg.lam, iters, r=cfg.r)
    dt = time.perf_counter() - t0
    rate_sample = iters / dt
    rate_full = rate_sample * (ks * ks) / (cfg.n * cfg.m)
    # oracle direct-sum throughput (pair evaluations/s of the matvec checks)
    kr = min(512, xs.shape[0])
    t0 = time.perf_counter()
    dense.direct_sum(xs[:kr], ys, bs, cfg.lam, 0, r=cfg.r)
    global ORACLE_PAIRS_PER_S
    ORACLE_PAIRS_PER_S = kr * ys.shape[0] / (time.perf_counter() - t0)
    desc = (f"{iters} log-domain Alg. 1 iterations on the first {ks}+{ks} points of {cfg.name} "
            f"({dt:.1f} s); value = sample it/s x ({ks}*{ks})/({cfg.n}*{cfg.m}) (quadratic extrapolation "
            f"to the full workload)")
    return rate_full, desc, dense.num_threads(), rate_sample


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    if args.steps is None:
        args.steps = 3
    cfg = get(args.config)
    from oracle import dense
    dense.build()
    for _ in range(max(args.warmup, 0) and 1):
        cpu_oracle_rate(cfg, 2.0)
    vals = []
    descs = []
    for _ in range(args.steps):
        v, desc, cores, _ = cpu_oracle_rate(cfg, args.cpu_seconds)
        vals.append(v)
        descs.append(desc)
    value = float(statistics.median(vals))
    line = {
        "impl": "reference", "metric": "sinkhorn_iterations_per_s", "value": value, "unit": "it/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
        "ms_per_step": 1e3 * cfg.iters / value, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": dict(workload_config(cfg), parallelism="host cores (CPU oracle, no GPU)"),
        "cpu_baseline": {"value": value, "unit": "it/s", "cores": cores, "kind": "oracle", "sample": descs[-1],
                         "cpu_model": cpu_model(), "nproc": os.cpu_count(),
                         "direct_sum_pair_evals_per_s": ORACLE_PAIRS_PER_S},
        "e2e": {"value": value, "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------- GPU arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    from paper_2201_07524_b200 import capi

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or args.nccl_self:
        # NCCL prints one "comm ... rank r nranks N ... Init COMPLETE" line per communicator on
        # stderr, so the ranks of both the torch and the library communicator can be checked
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = get(args.config)
    x, y, a, b = make_inputs(cfg)
    lo, hi = shard_range(cfg.n, rank, world)
    lo2, hi2 = shard_range(cfg.m, rank, world)
    hx, ha = np.ascontiguousarray(x[lo:hi]), np.ascontiguousarray(a[lo:hi])
    hy, hb = np.ascontiguousarray(y[lo2:hi2]), np.ascontiguousarray(b[lo2:hi2])
    del x, y, a, b
    dev = lambda z: torch.from_numpy(z).cuda()  # noqa: E731
    dx, dy, da, db = dev(hx), dev(hy), dev(ha), dev(hb)
    stream = torch.cuda.current_stream()
    if world > 1:
        ctx = capi.init_distributed_context(local, stream)
    elif args.nccl_self:
        ctx = capi.Context(local, 0, 1, capi.sk_nccl_unique_id(), stream)
    else:
        ctx = capi.Context(local, stream=stream)
    def solve_r1(x_, y_, a_, b_):
        """r = 1 workloads (NEXT-2): the same step through the C-ABI calls sinkhorn_solve wraps
        for r = 2 (fastsum_plan_ex with the Laplace kernel + near field, Alg. 2, divergences)."""
        P = capi.Plan(ctx, x_, y_, cfg.lam, cfg.N, cfg.sigma, cfg.m_w, cfg.eps_B, cfg.p, r=1,
                      near_cells=cfg.near_cells)
        u, v, info = capi.sinkhorn_run(P, a_, b_, cfg.iters)
        sd, sc = capi.sinkhorn_divergence(P, a_, b_, u, v)
        P.close()
        return sd, sc, info

    if cfg.r == 1:
        solve = lambda: solve_r1(dx, dy, da, db)  # noqa: E731
    else:
        solve = lambda: capi.sinkhorn_solve(ctx, dx, dy, da, db, cfg.lam, cfg.N, cfg.sigma, cfg.m_w,  # noqa: E731
                                            cfg.eps_B, cfg.p, cfg.iters)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")   # 256 MB > L2

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        solve()
    torch.cuda.synchronize()
    if args.steps is None:
        # launch/latency-bound small workloads: time enough steps (~1.5 s) that host and clock
        # transients average out; the same K on every rank
        t0 = time.perf_counter()
        solve()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        k = torch.tensor([max(3, min(200, int(1.5 / max(dt, 1e-4))))], dtype=torch.int64, device="cuda")
        if world > 1:
            dist.all_reduce(k, op=dist.ReduceOp.MIN)
        args.steps = int(k.item())

    # ---- timed region: K steps on HBM-resident inputs, L2 flushed between steps
    clocks = ClockSampler(local)
    clocks.start()
    # the timed steps run the product path (Sinkhorn iterations replayed as CUDA graphs); the
    # per-stage CUDA-event profile comes from one extra profiled step below
    capi.sk_profile(False)
    launches0 = capi.sk_launch_count()
    total_ms = 0.0
    results = None
    for _ in range(args.steps):
        flush.fill_(1.0)
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        results = solve()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        total_ms += e0.elapsed_time(e1)
    launches = capi.sk_launch_count() - launches0
    clk = clocks.stop()
    # ---- stage profile: one more step with CUDA events around every stage on the library
    # stream (graph replay off while profiling), same inputs, right after the timed region
    prof, prof_step_ms = {}, None
    if STAGE_PROFILE:
        flush.fill_(1.0)
        torch.cuda.synchronize()
        capi.sk_profile(True)
        capi.sk_profile_read(reset=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        solve()
        e1.record(stream)
        torch.cuda.synchronize()
        prof_step_ms = e0.elapsed_time(e1)
        prof = capi.sk_profile_read(reset=True)
        capi.sk_profile(False)
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    value = args.steps * cfg.iters / (total_ms * 1e-3)

    # ---- e2e: same step through the C-ABI with pinned HOST buffers (H2D + D2H inside)
    e2e = None
    if not args.no_e2e:
        pin = lambda z: torch.from_numpy(z).pin_memory()  # noqa: E731
        px, py, pa, pb = pin(hx), pin(hy), pin(ha), pin(hb)
        if cfg.r == 1:   # host buffers: the copies to the device are part of the step
            solve_h = lambda: solve_r1(px.cuda(non_blocking=True), py.cuda(non_blocking=True),  # noqa: E731
                                       pa.cuda(non_blocking=True), pb.cuda(non_blocking=True))
        else:
            solve_h = lambda: capi.sinkhorn_solve(ctx, px, py, pa, pb, cfg.lam, cfg.N, cfg.sigma, cfg.m_w,  # noqa
                                                  cfg.eps_B, cfg.p, cfg.iters, inputs_on_host=True)
        solve_h()
        tot = 0.0
        for _ in range(args.steps):
            flush.fill_(1.0)
            barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            solve_h()
            e1.record(stream)
            torch.cuda.synchronize()
            barrier()
            tot += e0.elapsed_time(e1)
        t = torch.tensor([tot], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        h2d = 8 * (hx.size + hy.size + ha.size + hb.size)
        e2e = {"value": args.steps * cfg.iters / (float(t.item()) * 1e-3), "unit": "it/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": 16}

    # ---- fast-summation point-evaluations/s: per direction, median over reps of
    # one fast summation each (CUDA events), max over ranks; also NUFFT points/s = (n_s + n_t)/t
    plan = capi.Plan(ctx, dx, dy, cfg.lam, cfg.N, cfg.sigma, cfg.m_w, cfg.eps_B, cfg.p, r=cfg.r,
                     near_cells=cfg.near_cells)
    box_size = plan.info()["box_size"]
    wy = torch.rand(hy.shape[0], dtype=torch.float64, device="cuda")
    wx = torch.rand(hx.shape[0], dtype=torch.float64, device="cuda")
    ox = torch.empty(hx.shape[0], dtype=torch.float64, device="cuda")
    oy = torch.empty(hy.shape[0], dtype=torch.float64, device="cuda")
    reps = 20 if cfg.n + cfg.m <= 2e7 else 5
    apply_dir = {}
    for tr, (w_, o_) in ((0, (wy, ox)), (1, (wx, oy))):
        for _ in range(2):
            capi.fastsum_apply(plan, w_, tr, 0, o_)
        torch.cuda.synchronize()
        times = []
        for _ in range(reps):
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            capi.fastsum_apply(plan, w_, tr, 0, o_)
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        t = torch.tensor([statistics.median(times)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        apply_dir[tr] = float(t.item())
    plan.close()
    apply_ms = apply_dir[0]
    point_evals = cfg.n / (apply_ms * 1e-3)

    # ---- roofline of the dominant kernel (from the live CUDA-event stage profile)
    pk = peaks()
    stage_ms = {s: (c, ms) for s, (c, ms) in prof.items() if c > 0}
    dom = max(("spread", "interp", "nearfield"), key=lambda s: stage_ms.get(s, (0, 0.0))[1])
    cnt, ms = stage_ms.get(dom, (1, float("nan")))
    avg_ms = ms / max(cnt, 1)
    W = 2 * cfg.m_w
    # per launch: spread/interp alternate between the x (n) and y (m) node sets -> mean (n+m)/2
    pts_per_launch = (cfg.n + cfg.m) / 2 / world
    flops = 2.0 * W ** cfg.d * pts_per_launch                 # one multiply-add per grid tap
    near_pairs, near_rad = None, None
    if cfg.r == 1 and cfg.d == 1 and world == 1:
        # NEXT-2 near field: exact pairs within the radius a = near_cells / (sigma N) torus units
        # (a / rho in the caller's units), counted on the host; the same count both directions
        Pq = capi.Plan(ctx, dx, dy, cfg.lam, cfg.N, cfg.sigma, cfg.m_w, cfg.eps_B, cfg.p, r=1,
                       near_cells=cfg.near_cells)
        near_rad = cfg.near_cells / (cfg.N * cfg.sigma) / Pq.info()["rho"]
        Pq.close()
        ys = np.sort(hy[:, 0])
        near_pairs = int((np.searchsorted(ys, hx[:, 0] + near_rad, side="left")
                          - np.searchsorted(ys, hx[:, 0] - near_rad, side="right")).sum())
    if dom == "nearfield":
        # per pair within the radius: |x - y|, r^2, (r/a)^2 (3), K_I Horner (p - 1 FMA), the
        # factored exp product (1), w (K - K_I) (1 FMA) and the accumulate (1): 2p + 5 flops
        flops = (2.0 * cfg.p + 5.0) * near_pairs
    sm_mhz = clk.get("sm_mhz") or pk.get("sm_max_mhz", 1965.0)
    fp64_peak = N_SM * FP64_FMA_PER_CLK_PER_SM * 2 * pk.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
    achieved = flops / (avg_ms * 1e-3) / 1e12
    bytes_alg = pts_per_launch * 8 * (cfg.d + 1) + (cfg.N * cfg.sigma) ** cfg.d * 8
    step_ms = total_ms / args.steps
    stage_share = {s: round(v[1] / prof_step_ms, 4) for s, v in stage_ms.items()} if prof_step_ms else {}
    G = (cfg.N * cfg.sigma) ** cfg.d
    n_avg = (cfg.n + cfg.m) / 2 / world
    alg_bytes = {"spread": n_avg * (cfg.d + 1) * 8 + G * 8, "interp": G * 8 + n_avg * (8 * cfg.d + 24),
                 "fft_fwd": 2 * G * 8, "fft_inv": 2 * G * 8}
    stage_hbm = {}
    for st_name, by in alg_bytes.items():
        c_, ms_ = stage_ms.get(st_name, (0, 0.0))
        if c_ > 0 and ms_ > 0:
            stage_hbm[st_name] = {"alg_bytes_per_launch": by, "avg_launch_ms": ms_ / c_,
                                  "frac": by / (ms_ / c_ * 1e-3) / (pk["hbm_gbs"] * 1e9)}
    traffic, traffic_src, traffic_note = None, None, None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            tr = json.load(fh).get(cfg.name, {}).get(dom)
        if tr and world == 1:
            traffic, traffic_src = float(tr["bytes_per_launch"]), tr["measured"]
            traffic_note = tr.get("note")
    except (OSError, ValueError, KeyError):
        pass
    line = {
        "metric": "sinkhorn_iterations_per_s", "value": value, "unit": "it/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generators of BASELINE.json configs; see DESIGN.md input recipe)",
        "config": {**workload_config(cfg),
                   "parallelism": f"dp{world} (point shards + grid all-reduce)"
                                  + (", one-rank NCCL communicator" if args.nccl_self and world == 1 else ""),
                   "l2": "256 MB buffer written between timed steps"},
        "fastsum_point_evals_per_s": point_evals,   # all n targets of one K v, max-over-ranks time
        "fastsum_apply_ms": apply_ms,
        "fastsum": {"Kv": {"ms": apply_dir[0], "point_evals_per_s": cfg.n / (apply_dir[0] * 1e-3),
                           "nufft_points_per_s": (cfg.n + cfg.m) / (apply_dir[0] * 1e-3)},
                    "KTu": {"ms": apply_dir[1], "point_evals_per_s": cfg.m / (apply_dir[1] * 1e-3),
                            "nufft_points_per_s": (cfg.n + cfg.m) / (apply_dir[1] * 1e-3)},
                    "reps": reps, "statistic": "median"},
        "roofline": {"bound": "alu", "kernel": dom, "achieved": achieved, "peak": fp64_peak,
                     "unit": "TFLOP/s", "frac": achieved / fp64_peak, "traffic": traffic,
                     "traffic_source": traffic_src,
                     "traffic_note": traffic_note,
                     # measured DRAM bytes (ncu) over the live launch time: how close the kernel's real
                     # traffic runs to the HBM roof
                     "traffic_hbm_frac": (traffic / (avg_ms * 1e-3) / (pk["hbm_gbs"] * 1e9)) if traffic else None,
                     "algorithmic": (f"2p + 5 = {2 * cfg.p + 5} flops per pair within the radius, {near_pairs} pairs/launch"
                                     if dom == "nearfield" else
                                     f"2*(2m_w)^d flops per node per launch, {pts_per_launch:.3g} nodes/launch"),
                     "peak_source": f"{N_SM} SMs x {FP64_FMA_PER_CLK_PER_SM} FP64 FMA/clk x 2 x sm_max_mhz "
                                    f"{pk.get('sm_max_mhz')} (DESIGN.md)",
                     "hbm_frac": bytes_alg / (avg_ms * 1e-3) / (pk["hbm_gbs"] * 1e9),
                     # what the kernel's FP64 instruction mix allows on this chip: the
                     # spread's 28-tile m8n8k4 cover issues 1792 DMMA FMAs + 256 DMUL lane products per
                     # node for 1728 useful FMAs on the one shared FP64 pipe (pipe model: 0.844 x
                     # 37.2 TF); the interp pays one DFMA per E value (microbenchmark of the same mix);
                     # d = 3, m_w = 6 only
                     "mix_ceiling_tflops": (MIX_CEILING.get(dom) if (cfg.d == 3 and cfg.m_w == 6) else None),
                     "frac_of_mix_ceiling": ((achieved / MIX_CEILING[dom])
                                             if (cfg.d == 3 and cfg.m_w == 6 and dom in MIX_CEILING) else None),
                     "mix_ceiling_source": "spread: pipe model 1728 / (1792 + 256) x 37.2 TF (DESIGN.md §6); "
                                           "interp: profiles/r1_interp_mix.txt (measured)",
                     "avg_launch_ms": avg_ms,
                     "timing": "CUDA events around the kernel's stage on the library stream, averaged "
                               "over its launches in the profiled step (stage_profile)"},
        "plan_ms_per_step": stage_ms.get("plan", (0, 0.0))[1],
        "stage_profile": {"how": "one extra step after the timed region with CUDA events around every "
                                 "stage on the library stream (graph replay off while profiling)",
                          "step_ms": prof_step_ms,
                          "stage_ms": {s: v[1] for s, v in stage_ms.items()},
                          "launches": {s: v[0] for s, v in stage_ms.items()}},
        "stage_share_of_step": stage_share,
        # SURVEY §8(d) per-stage HBM fraction (BJ metric "% HBM roofline for the spread, FFT and
        # interpolate stages"): algorithmic bytes per launch / measured launch time / HBM peak.
        # spread: n_s (d+1) 8 + G 8; interp: G 8 + n_t (8d + 24); FFT: 2 G 8 per transform (full
        # grid; the pruned d = 3 path moves less than this definition charges)
        "stage_hbm_frac": stage_hbm,
        "gpu_launches": int(launches),
        "comm": {"world": world, "rank0_of": world,
                 "backend": "nccl" if (world > 1 or args.nccl_self) else "none (one rank)",
                 "grid_allreduce_bytes_per_apply": (8 * box_size if (world > 1 or args.nccl_self) else 0),
                 "collective": "ncclAllReduce(sum, f64) of the touched grid box per fast summation "
                               "+ scalar all-reduces (DESIGN.md §7)"},
        "spread_mode": "deterministic (fixed-point)" if os.environ.get("SK_DETERMINISTIC", "1") != "0" else "fp64 atomics",
        "clocks": clk,
        "divergence": {"s_dual": results[0], "s_cost": results[1]} if results else None,
        "kappa_log10_est": results[2].kappa_log10_est if results else None,
        # SURVEY §8(d)'s narrower definition: iterations / device time of sinkhorn_run alone
        # (no plan, no divergence), from the run's own CUDA events, last timed step, rank 0
        "sinkhorn_run_iterations_per_s": (cfg.iters / results[2].seconds) if results and results[2].seconds > 0 else None,
    }
    if near_pairs is not None:
        c_n, ms_n = stage_ms.get("nearfield", (0, 0.0))
        nf_ms = ms_n / max(c_n, 1)
        line["nearfield"] = {"radius_caller_units": near_rad, "pairs_per_apply": near_pairs,
                             "avg_launch_ms": nf_ms,
                             "pair_evals_per_s": near_pairs / (nf_ms * 1e-3) if ms_n else None,
                             "flops_per_pair": 2 * cfg.p + 5,
                             "note": "position-sorted nodes, 32 targets x 8 warps per CTA over the contiguous "
                                     "source range in the radius, factored exp (DESIGN.md §9b)"}
    if e2e:
        line["e2e"] = e2e
    if rank == 0 and world == 1 and not args.no_cpu_baseline:   # the oracle baseline: rank 0 at N = 1 only
        v, desc, cores, _ = cpu_oracle_rate(cfg, args.cpu_seconds)
        line["cpu_baseline"] = {"value": v, "unit": "it/s", "cores": cores, "kind": "oracle", "sample": desc,
                                "cpu_model": cpu_model(), "nproc": os.cpu_count(),
                                "direct_sum_pair_evals_per_s": ORACLE_PAIRS_PER_S}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
