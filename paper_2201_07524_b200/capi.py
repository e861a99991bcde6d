"""Thin ctypes binding of libsk_nfft.so (include/sinkhorn_nfft.h). Argument marshalling only:
every step of the hot path runs in the library's CUDA kernels. There is no CPU fallback --
importing this module raises if the in-tree library is missing.

Tensors must be CUDA float64, contiguous, on the context's device (except where a host array
is documented). Names mirror the C entry points.
"""
from __future__ import annotations

import ctypes
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SK_LIB_PATH") or os.path.join(_PKG, "lib", "libsk_nfft.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libsk_nfft.so not built ({LIB_PATH}); run `python -m paper_2201_07524_b200.build` "
                      "or __graft_entry__.build()")

_lib = ctypes.CDLL(LIB_PATH)

_vp = ctypes.c_void_p
_i = ctypes.c_int
_ll = ctypes.c_longlong
_d = ctypes.c_double
_dp = ctypes.POINTER(ctypes.c_double)

SK_OK, SK_EINVAL, SK_EGEOMETRY, SK_ENONPOS, SK_ENOTCONVERGED, SK_ECUDA, SK_ECUFFT, SK_ENCCL, SK_ENOMEM = range(9)
_NAMES = {0: "SK_OK", 1: "SK_EINVAL", 2: "SK_EGEOMETRY", 3: "SK_ENONPOS", 4: "SK_ENOTCONVERGED",
          5: "SK_ECUDA", 6: "SK_ECUFFT", 7: "SK_ENCCL", 8: "SK_ENOMEM"}


class PlanOpts(ctypes.Structure):
    _fields_ = [("lam", ctypes.c_double), ("r", ctypes.c_int), ("N", ctypes.c_int), ("sigma", ctypes.c_double),
                ("m_w", ctypes.c_int), ("eps_B", ctypes.c_double), ("p_smooth", ctypes.c_int),
                ("near_cells", ctypes.c_int)]


class RunInfo(ctypes.Structure):
    _fields_ = [("iters_done", ctypes.c_int), ("residual", ctypes.c_double), ("bad_iter", ctypes.c_int),
                ("bad_index", ctypes.c_longlong), ("kappa_log10_est", ctypes.c_double),
                ("seconds", ctypes.c_double), ("kappa_u_log10_est", ctypes.c_double), ("bad_side", ctypes.c_int),
                ("bad_rank", ctypes.c_int)]

    def asdict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class SkError(RuntimeError):
    def __init__(self, code, msg, info=None):
        super().__init__(f"{_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.info = info


_sig = {
    "sinkhorn_init": ([ctypes.POINTER(_vp), _i, _i, _i, _vp, _vp], _i),
    "sinkhorn_finalize": ([_vp], _i),
    "sk_nccl_unique_id": ([_vp], _i),
    "fastsum_plan": ([_vp, ctypes.POINTER(_vp), _i, _vp, _ll, _vp, _ll, _d, _i, _d, _i, _d, _i], _i),
    "fastsum_plan_ex": ([_vp, ctypes.POINTER(_vp), _i, _vp, _ll, _vp, _ll, ctypes.POINTER(PlanOpts)], _i),
    "fastsum_plan_destroy": ([_vp], _i),
    "fastsum_apply": ([_vp, _i, _i, _vp, _vp], _i),
    "sinkhorn_run": ([_vp, _vp, _vp, _i, _d, _i, _vp, _vp, ctypes.POINTER(RunInfo)], _i),
    "sinkhorn_run_trace": ([_vp, _vp, _vp, _i, _d, _i, _vp, _vp, ctypes.POINTER(RunInfo), _dp], _i),
    "sinkhorn_divergence": ([_vp, _vp, _vp, _vp, _vp, _dp, _dp], _i),
    "sinkhorn_solve": ([_vp, _i, _vp, _ll, _vp, _ll, _vp, _vp, _d, _i, _d, _i, _d, _i, _i, _i, _dp, _dp,
                        ctypes.POINTER(RunInfo)], _i),
    "nfft_spread": ([_vp, _i, _vp, _vp], _i),
    "nfft_interp": ([_vp, _i, _vp, _vp], _i),
    "fastsum_plan_info": ([_vp, _dp], _i),
    "fastsum_coefficients": ([_vp, _i, _dp], _i),
    "sk_launch_count": ([], _ll),
    "sk_release_cache": ([], None),
    "sk_profile": ([_i], None),
    "sk_profile_read": ([_dp, _i, _i], _i),
    "sk_last_error": ([], ctypes.c_char_p),
}
for _name, (_args, _res) in _sig.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res

EXPORTED = tuple(_sig.keys())


def _check(code, info=None):
    if code != SK_OK:
        raise SkError(code, _lib.sk_last_error().decode(errors="replace"), info)


def _ptr(t):
    if t is None:
        return None
    if not isinstance(t, torch.Tensor):
        raise TypeError("expected a torch tensor")
    if not t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
        raise ValueError("expected a contiguous CUDA float64 tensor")
    return ctypes.c_void_p(t.data_ptr()) if t.numel() else None


def _ptr_n(t, n, what):
    """_ptr with a length check against the plan's node count (the library trusts lengths)."""
    if t is not None and t.numel() != n:
        raise ValueError(f"{what}: expected {n} elements, got {t.numel()}")
    return _ptr(t)


def _hptr(a):
    """Host numpy float64 C-contiguous array (or pinned CPU tensor) -> pointer."""
    if isinstance(a, torch.Tensor):
        assert a.device.type == "cpu" and a.dtype == torch.float64 and a.is_contiguous()
        return ctypes.c_void_p(a.data_ptr()) if a.numel() else None
    assert a.dtype.name == "float64" and a.flags["C_CONTIGUOUS"]
    return ctypes.c_void_p(a.ctypes.data) if a.size else None


def sk_launch_count() -> int:
    return int(_lib.sk_launch_count())


STAGES = ("spread", "allreduce", "fft_fwd", "multiply", "fft_inv", "interp", "update", "plan", "nearfield")


def sk_profile(on: bool) -> None:
    _lib.sk_profile(1 if on else 0)


def sk_profile_read(reset: bool = True) -> dict:
    """{stage: (timed launches, total device ms)} from the library's CUDA-event profiler."""
    out = (ctypes.c_double * (2 * len(STAGES)))()
    _check(_lib.sk_profile_read(out, len(STAGES), 1 if reset else 0))
    return {s: (int(out[2 * k]), float(out[2 * k + 1])) for k, s in enumerate(STAGES)}


def sk_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.sk_nccl_unique_id(ctypes.cast(buf, _vp)))
    return buf.raw


class Context:
    """sinkhorn_init / sinkhorn_finalize. stream: torch.cuda.Stream (default: current)."""

    def __init__(self, device: int = 0, rank: int = 0, world_size: int = 1, nccl_id: bytes | None = None,
                 stream: torch.cuda.Stream | None = None):
        torch.cuda.set_device(device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        self.device = device
        self.rank, self.world_size = rank, world_size
        h = _vp()
        idbuf = None if nccl_id is None else ctypes.create_string_buffer(nccl_id, 128)
        _check(_lib.sinkhorn_init(ctypes.byref(h), device, rank, world_size,
                                  None if idbuf is None else ctypes.cast(idbuf, _vp),
                                  _vp(self.stream.cuda_stream)))
        self.handle = h

    def close(self):
        if self.handle:
            _lib.sinkhorn_finalize(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def init_distributed_context(device: int, stream=None) -> Context:
    """SPMD helper: rank 0 creates the ncclUniqueId, torch.distributed broadcasts it."""
    import torch.distributed as dist
    rank, world = dist.get_rank(), dist.get_world_size()
    if world == 1:
        return Context(device, 0, 1, None, stream)
    obj = [sk_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return Context(device, rank, world, obj[0], stream)


class Plan:
    """fastsum_plan / fastsum_plan_destroy (x: [n, d], y: [m, d] CUDA float64)."""

    def __init__(self, ctx: Context, x: torch.Tensor, y: torch.Tensor, lam: float, N: int, sigma: float = 2.0,
                 m_w: int = 8, eps_B: float = 1 / 16, p_smooth: int = 8, r: int = 2, near_cells: int = 16):
        """r = 2: fastsum_plan; r = 1: fastsum_plan_ex (Laplace kernel + near field)."""
        d = x.shape[1] if x.dim() == 2 else 1
        self.ctx, self.d = ctx, d
        self.n, self.m = x.shape[0], y.shape[0]
        self.lam, self.r = lam, r
        h = _vp()
        if r == 2:
            _check(_lib.fastsum_plan(ctx.handle, ctypes.byref(h), d, _ptr(x), self.n, _ptr(y), self.m, float(lam),
                                     int(N), float(sigma), int(m_w), float(eps_B), int(p_smooth)))
        else:
            o = PlanOpts(float(lam), int(r), int(N), float(sigma), int(m_w), float(eps_B), int(p_smooth),
                         int(near_cells))
            _check(_lib.fastsum_plan_ex(ctx.handle, ctypes.byref(h), d, _ptr(x), self.n, _ptr(y), self.m,
                                        ctypes.byref(o)))
        self.handle = h
        info = self.info()
        self.grid_n = int(info["n_grid"])

    def close(self):
        if self.handle:
            _lib.fastsum_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> dict:
        out = (ctypes.c_double * 22)()
        _check(_lib.fastsum_plan_info(self.handle, out))
        return dict(centre=list(out[0:3]), rho=out[3], lambda_p=out[4], L=out[5], n_grid=out[6],
                    band=out[7], d=out[8], total_x=out[9], total_y=out[10],
                    box_lo=[int(v) for v in out[11:14]], box_n=[int(v) for v in out[14:17]],
                    box_size=int(out[17]), band_tail=(out[18], out[19]), K_at_L=out[20],
                    gauss_trunc=out[21])

    def coefficients(self, kernel: int = 0):
        import numpy as np
        nb = int(self.info()["band"])
        b = np.empty((nb,) * self.d)
        _check(_lib.fastsum_coefficients(self.handle, kernel, b.ctypes.data_as(_dp)))
        return b


def fastsum_apply(plan: Plan, w: torch.Tensor, transpose: int = 0, kernel: int = 0, out=None):
    """transpose 0: t = K w (w on y, t on x); 1: t = K^T w. kernel 0: exp(-lam c); 1: c exp(-lam c)."""
    cnt = plan.m if transpose else plan.n
    t = out if out is not None else torch.empty(cnt, dtype=torch.float64, device=w.device)
    _check(_lib.fastsum_apply(plan.handle, int(transpose), int(kernel), _ptr_n(w, plan.n if transpose else plan.m, "w"),
                              _ptr_n(t, cnt, "t")))
    return t


def nfft_spread(plan: Plan, side: int, w: torch.Tensor):
    g = torch.empty((plan.grid_n,) * plan.d, dtype=torch.float64, device=w.device)
    _check(_lib.nfft_spread(plan.handle, int(side), _ptr_n(w, plan.n if side == 0 else plan.m, "w"), _ptr(g)))
    return g


def nfft_interp(plan: Plan, side: int, grid: torch.Tensor):
    cnt = plan.n if side == 0 else plan.m
    t = torch.empty(cnt, dtype=torch.float64, device=grid.device)
    _check(_lib.nfft_interp(plan.handle, int(side), _ptr_n(grid.contiguous(), plan.grid_n ** plan.d, "grid"), _ptr(t)))
    return t


def sinkhorn_run(plan: Plan, a, b, iters: int, tol: float = 0.0, rescale_policy: int = 0, u=None, v=None):
    """Alg. 2; returns (u, v, RunInfo). u, v default to all-ones (cold start)."""
    u = torch.ones(plan.n, dtype=torch.float64, device=a.device) if u is None else u
    v = torch.ones(plan.m, dtype=torch.float64, device=a.device) if v is None else v
    info = RunInfo()
    code = _lib.sinkhorn_run(plan.handle, _ptr_n(a, plan.n, "a"), _ptr_n(b, plan.m, "b"), int(iters), float(tol),
                             int(rescale_policy), _ptr_n(u, plan.n, "u"), _ptr_n(v, plan.m, "v"), ctypes.byref(info))
    _check(code, info)
    return u, v, info


TRACE_FIELDS = ("row_resid", "row_kl", "sum_a_log_u", "col_resid", "col_kl", "sum_b_log_v")


def sinkhorn_run_trace(plan: Plan, a, b, iters: int, tol: float = 0.0, rescale_policy: int = 0, u=None, v=None):
    """Alg. 2 with per-iteration diagnostics; returns (u, v, RunInfo, trace [iters, 6] numpy,
    columns TRACE_FIELDS; NaN rows for iterations not run)."""
    import numpy as np
    u = torch.ones(plan.n, dtype=torch.float64, device=a.device) if u is None else u
    v = torch.ones(plan.m, dtype=torch.float64, device=a.device) if v is None else v
    info = RunInfo()
    tr = np.empty((max(int(iters), 0), 6))
    code = _lib.sinkhorn_run_trace(plan.handle, _ptr_n(a, plan.n, "a"), _ptr_n(b, plan.m, "b"), int(iters),
                                   float(tol), int(rescale_policy), _ptr_n(u, plan.n, "u"), _ptr_n(v, plan.m, "v"),
                                   ctypes.byref(info), tr.ctypes.data_as(_dp))
    _check(code, info)
    return u, v, info, tr


def sinkhorn_divergence(plan: Plan, a, b, u, v):
    """Returns (s_dual, s_cost)."""
    sd, sc = ctypes.c_double(), ctypes.c_double()
    _check(_lib.sinkhorn_divergence(plan.handle, _ptr_n(a, plan.n, "a"), _ptr_n(b, plan.m, "b"),
                                    _ptr_n(u, plan.n, "u"), _ptr_n(v, plan.m, "v"), ctypes.byref(sd), ctypes.byref(sc)))
    return sd.value, sc.value


def sinkhorn_solve(ctx: Context, x, y, a, b, lam, N, sigma=2.0, m_w=8, eps_B=1 / 16, p_smooth=8, iters=100,
                   inputs_on_host: bool = False):
    """Plan + Alg. 2 + divergences in one C call. Host arrays (numpy / pinned CPU tensors) when
    inputs_on_host, else CUDA tensors. Returns (s_dual, s_cost, RunInfo)."""
    d = x.shape[1] if len(x.shape) == 2 else 1
    P = _hptr if inputs_on_host else _ptr
    sd, sc = ctypes.c_double(), ctypes.c_double()
    info = RunInfo()
    code = _lib.sinkhorn_solve(ctx.handle, d, P(x), x.shape[0], P(y), y.shape[0], P(a), P(b), float(lam), int(N),
                               float(sigma), int(m_w), float(eps_B), int(p_smooth), int(iters),
                               1 if inputs_on_host else 0, ctypes.byref(sd), ctypes.byref(sc), ctypes.byref(info))
    _check(code, info)
    return sd.value, sc.value, info
