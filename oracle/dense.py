"""ctypes front-end of oracle.c (dense FP64 direct sums and Alg. 1). TEST INFRASTRUCTURE.

See oracle.c's header for the paper passages each routine follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_D = ctypes.POINTER(ctypes.c_double)
_LL = ctypes.POINTER(ctypes.c_longlong)


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (plain -O2, OpenMP, portable x86-64)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", _SRC, "-o", _LIB, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.oracle_direct_sum.argtypes = [ctypes.c_int, _D, ctypes.c_longlong, _D, ctypes.c_longlong,
                                        _D, ctypes.c_double, ctypes.c_int, ctypes.c_int, _LL, ctypes.c_longlong, _D]
        L.oracle_sinkhorn_plain.argtypes = [ctypes.c_int, _D, ctypes.c_longlong, _D, ctypes.c_longlong,
                                            _D, _D, ctypes.c_double, ctypes.c_int, ctypes.c_int, _D, _D]
        L.oracle_sinkhorn_plain.restype = ctypes.c_int
        L.oracle_sinkhorn_log.argtypes = [ctypes.c_int, _D, ctypes.c_longlong, _D, ctypes.c_longlong,
                                          _D, _D, ctypes.c_double, ctypes.c_int, ctypes.c_int, _D, _D, _D]
        L.oracle_divergence.argtypes = [ctypes.c_int, _D, ctypes.c_longlong, _D, ctypes.c_longlong,
                                        _D, _D, ctypes.c_double, ctypes.c_int, _D, _D, _D]
        L.oracle_num_threads.restype = ctypes.c_int
        L.oracle_set_threads.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(_D)


def _c(a, dtype=np.float64):
    return np.ascontiguousarray(a, dtype=dtype)


def num_threads() -> int:
    return lib().oracle_num_threads()


def set_threads(nt: int) -> None:
    lib().oracle_set_threads(int(nt))


def direct_sum(x, y, w, lam, kernel=0, rows=None, r=2):
    """t_i = sum_j w_j K(x_i, y_j), K = exp(-lam c) (kernel 0) or c exp(-lam c) (kernel 1),
    c = |x_i - y_j|^r (r = 2 or 1). Eq. (matexp); transpose (matexpt) = swap x
    and y. ``rows`` restricts to a subset of target rows (returned in that order)."""
    x = _c(x).reshape(len(x), -1)
    y = _c(y).reshape(len(y), -1)
    w = _c(w)
    d = x.shape[1]
    assert y.shape[1] == d and w.shape[0] == y.shape[0]
    if rows is None:
        out = np.empty(x.shape[0])
        lib().oracle_direct_sum(d, _p(x), x.shape[0], _p(y), y.shape[0], _p(w), float(lam), int(r),
                                int(kernel), None, 0, _p(out))
    else:
        rows = _c(rows, np.int64)
        out = np.empty(rows.shape[0])
        lib().oracle_direct_sum(d, _p(x), x.shape[0], _p(y), y.shape[0], _p(w), float(lam), int(r),
                                int(kernel), rows.ctypes.data_as(_LL), rows.shape[0], _p(out))
    return out


def sinkhorn_plain(x, y, a, b, lam, iters, r=2):
    """Alg. 1 literally in the scaling domain; returns (alpha, alpha~, n_bad)."""
    x = _c(x).reshape(len(x), -1)
    y = _c(y).reshape(len(y), -1)
    a, b = _c(a), _c(b)
    al, at = np.empty(x.shape[0]), np.empty(y.shape[0])
    bad = lib().oracle_sinkhorn_plain(x.shape[1], _p(x), x.shape[0], _p(y), y.shape[0], _p(a), _p(b),
                                      float(lam), int(r), int(iters), _p(al), _p(at))
    return al, at, bad


def sinkhorn_log(x, y, a, b, lam, iters, g0=None, r=2):
    """Alg. 1 in potentials f = log(alpha)/lam, g = log(alpha~)/lam (g^0 = 0, f first)."""
    x = _c(x).reshape(len(x), -1)
    y = _c(y).reshape(len(y), -1)
    a, b = _c(a), _c(b)
    f, g = np.empty(x.shape[0]), np.empty(y.shape[0])
    gin = None if g0 is None else _p(_c(g0))
    lib().oracle_sinkhorn_log(x.shape[1], _p(x), x.shape[0], _p(y), y.shape[0], _p(a), _p(b),
                              float(lam), int(r), int(iters), gin, _p(f), _p(g))
    return f, g


def divergence(x, y, a, b, lam, f, g, r=2):
    """dict(s_cost=s~, s_dual=s, mass, row_resid, col_resid, entropy) from potentials.
    Def 3.1, Eq. (14), Eq. (Error)."""
    x = _c(x).reshape(len(x), -1)
    y = _c(y).reshape(len(y), -1)
    a, b, f, g = _c(a), _c(b), _c(f), _c(g)
    out = np.empty(6)
    lib().oracle_divergence(x.shape[1], _p(x), x.shape[0], _p(y), y.shape[0], _p(a), _p(b),
                            float(lam), int(r), _p(f), _p(g), _p(out))
    return dict(s_cost=out[0], s_dual=out[1], mass=out[2], row_resid=out[3], col_resid=out[4],
                entropy=out[5])


def sinkhorn_divergence(x, y, a, b, lam, iters, r=2):
    """Convenience: log-domain Alg. 1 then divergences. Returns (dict, f, g)."""
    f, g = sinkhorn_log(x, y, a, b, lam, iters, r=r)
    return divergence(x, y, a, b, lam, f, g, r=r), f, g
