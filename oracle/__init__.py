"""ctypes binding of liboracle.so -- TEST INFRASTRUCTURE ONLY.

The oracle is the plain fp64 CPU implementation of the hot path of arXiv 1209.1910
(/root/reference/PAPER.md), written from the paper and pinned by tests/test_oracle_*.py
against closed forms, brute force and library routines.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this module.  The product package (paper_1209_1910_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liboracle.so")

EPS = 2.0 ** -53


def build(force: bool = False) -> str:
    """Compile liboracle.so with the oracle Makefile (no FMA contraction)."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE, "liboracle.so"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        D = C.POINTER(C.c_double)
        I64 = C.c_int64
        P = C.c_void_p
        sig = {
            "orc_tnorm": (C.c_double, [I64, P, P]),
            "orc_clusters": (I64, [I64, P, C.c_double, P]),
            "orc_shifts": (None, [I64, P, I64, P, P]),
            "orc_splitmix64": (C.c_uint64, [C.c_uint64, C.c_uint64]),
            "orc_rng_uniform": (C.c_double, [C.c_uint64, C.c_uint64]),
            "orc_start_vector": (None, [I64, C.c_uint64, I64, I64, P]),
            "orc_lu_factor": (None, [I64, P, P, C.c_double, C.c_double, P, P, P, P, P]),
            "orc_lu_solve": (None, [I64, P, P, P, P, P, P]),
            "orc_reflector": (C.c_double, [I64, P, P, D, D]),
            "orc_householder_orth": (None, [I64, I64, P, P]),
            "orc_cwy_orth": (None, [I64, I64, P, P]),
            "orc_cwy_ordinary_orth": (None, [I64, I64, P, P]),
            "orc_cwy_build": (None, [I64, I64, P, P]),
            "orc_cwy_apply_block": (None, [I64, I64, P, I64, P, C.c_int, P]),
            "orc_sturm_count": (I64, [I64, P, P, C.c_double, C.c_double]),
            "orc_bisect": (None, [I64, P, P, P]),
            "orc_eigvecs": (I64, [I64, P, P, P, P, I64, C.c_uint64, P]),
            "orc_eigvecs_range": (I64, [I64, P, P, P, P, I64, C.c_uint64, P, I64, I64]),
            "orc_eigvecs_mgs_range": (I64, [I64, P, P, P, P, I64, C.c_uint64, P, I64, I64]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _e(e, n):
    e = _f64(e if e is not None else np.zeros(0))
    if n > 1 and e.shape[0] != n - 1:
        raise ValueError("e must have n-1 entries")
    return e if n > 1 else np.zeros(1)


def tnorm(d, e):
    d = _f64(d)
    n = d.shape[0]
    return lib().orc_tnorm(n, _p(d), _p(_e(e, n)))


def clusters(w, tn):
    w = _f64(w)
    n = w.shape[0]
    cs = np.zeros(n + 1, dtype=np.int64)
    nc = lib().orc_clusters(n, _p(w), float(tn), _p(cs))
    return cs[: nc + 1].copy()


def shifts(w, cstart):
    w = _f64(w)
    cs = np.ascontiguousarray(cstart, dtype=np.int64)
    wt = np.zeros_like(w)
    lib().orc_shifts(w.shape[0], _p(w), cs.shape[0] - 1, _p(cs), _p(wt))
    return wt


def splitmix64(seed, ctr):
    return int(lib().orc_splitmix64(seed, ctr))


def rng_uniform(seed, ctr):
    return float(lib().orc_rng_uniform(seed, ctr))


def start_vector(n, seed, j, restart=0):
    b = np.zeros(n)
    lib().orc_start_vector(n, seed, j, restart, _p(b))
    return b


def lu_factor(d, e, shift, tn=None):
    d = _f64(d)
    n = d.shape[0]
    ee = _e(e, n)
    if tn is None:
        tn = tnorm(d, e)
    m1 = max(n - 1, 1)
    l = np.zeros(m1)
    piv = np.zeros(m1, dtype=np.int8)
    u0 = np.zeros(n)
    u1 = np.zeros(m1)
    u2 = np.zeros(max(n - 2, 1))
    lib().orc_lu_factor(n, _p(d), _p(ee), float(shift), float(tn), _p(l), _p(piv), _p(u0), _p(u1), _p(u2))
    return dict(l=l, piv=piv, u0=u0, u1=u1, u2=u2, n=n)


def lu_solve(f, b):
    x = _f64(b).copy()
    lib().orc_lu_solve(f["n"], _p(f["l"]), _p(f["piv"]), _p(f["u0"]), _p(f["u1"]), _p(f["u2"]), _p(x))
    return x


def reflector(u):
    u = _f64(u)
    y = np.zeros_like(u)
    c = C.c_double()
    t = C.c_double()
    nu = lib().orc_reflector(u.shape[0], _p(u), _p(y), C.byref(c), C.byref(t))
    return y, c.value, t.value, nu


def _orth(fn, V):
    V = np.asfortranarray(V, dtype=np.float64)
    n, m = V.shape
    Q = np.zeros((n, m), order="F")
    getattr(lib(), fn)(n, m, V.ctypes.data_as(C.c_void_p), Q.ctypes.data_as(C.c_void_p))
    return Q


def householder_orth(V):
    """Alg. 2, ordinary sign q_j = H_1..H_j e_j."""
    return _orth("orc_householder_orth", V)


def cwy_orth(V):
    """Alg. 3 in the §3.3.2 packed formulation (sign-flipped q)."""
    return _orth("orc_cwy_orth", V)


def cwy_ordinary_orth(V):
    """Alg. 3 in the §3.3.1 ordinary formulation (T_j erratum applied)."""
    return _orth("orc_cwy_ordinary_orth", V)


def cwy_build(V):
    """Packed Y/T buffer ((n+1) x m, column-major) after m §3.3.2 steps on V's columns.
    Returns (Y, T) unpacked: Y n x m lower trapezoidal, T m x m upper triangular."""
    V = np.asfortranarray(V, dtype=np.float64)
    n, m = V.shape
    P = np.zeros((n + 1, m), order="F")
    lib().orc_cwy_build(n, m, V.ctypes.data_as(C.c_void_p), P.ctypes.data_as(C.c_void_p))
    Y = np.zeros((n, m))
    T = np.zeros((m, m))
    for k in range(m):
        T[:k, k] = P[:k, k]
        T[k, k] = P[k, k]
        Y[k:, k] = P[k + 1:, k]
    return Y, T


def cwy_apply_block(V, X, trans=True):
    """Blocked look-ahead oracle: with Y, T from V's columns (§3.3.2),
    U = X - Y T^T Y^T X (trans) or X - Y T Y^T X."""
    V = np.asfortranarray(V, dtype=np.float64)
    X = np.asfortranarray(X, dtype=np.float64)
    n, k = V.shape
    b = X.shape[1]
    U = np.zeros((n, b), order="F")
    lib().orc_cwy_apply_block(n, k, V.ctypes.data_as(C.c_void_p), b, X.ctypes.data_as(C.c_void_p), int(bool(trans)),
                              U.ctypes.data_as(C.c_void_p))
    return U


def sturm_count(d, e, x, tn=None):
    d = _f64(d)
    n = d.shape[0]
    if tn is None:
        tn = tnorm(d, e)
    return int(lib().orc_sturm_count(n, _p(d), _p(_e(e, n)), float(x), float(tn)))


def bisect(d, e):
    d = _f64(d)
    n = d.shape[0]
    w = np.zeros(n)
    lib().orc_bisect(n, _p(d), _p(_e(e, n)), _p(w))
    return w


def eigvecs(d, e, w, seed=1, j_lo=0, j_hi=None, return_iters=False, mgs=False):
    """Alg. 4 (DSTEIN-cWY), or with mgs=True Alg. 1 (classical MGS
    reorthogonalisation).  Returns (Z, info[, iters]); Z is
    column-major n x (j_hi - j_lo) holding eigenvectors j_lo .. j_hi-1."""
    d = _f64(d)
    w = _f64(w)
    n = d.shape[0]
    if j_hi is None:
        j_hi = n
    # Z holds only columns [j_lo, j_hi); the C side addresses column j at Z0 + j*n.
    Z = np.zeros((n, j_hi - j_lo), order="F")
    iters = np.zeros(n, dtype=np.int32)
    z0 = C.c_void_p(Z.ctypes.data - 8 * n * int(j_lo))
    fn = lib().orc_eigvecs_mgs_range if mgs else lib().orc_eigvecs_range
    info = fn(n, _p(d), _p(_e(e, n)), _p(w), z0, n, int(seed), _p(iters), int(j_lo), int(j_hi))
    if return_iters:
        return Z, int(info), iters
    return Z, int(info)
