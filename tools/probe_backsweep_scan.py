"""Probe (CPU, numpy + the oracle's LU): why the chained solve's back substitution stays serial.

The back recurrence x_i = t_i - b_i x_{i+1} - c_i x_{i+2} (U = row-normalised upper factor of
T - w_j I, partial pivoting) is rerun here (a) serially and (b) in chunks of L rows whose
incoming state is carried from chunk to chunk through the chunk's 2x2 affine map (the
partitioned / scan formulation).  On the glued Wilkinson matrix (cfg3) the composed maps
cancel catastrophically -- relative errors of 1e-2 up to overflow even for L = 2 -- because the
homogeneous solutions grow by up to 1/eps at the near-singular pivot.  The forward
recurrence (|l_i| <= 1) has no such growth and is partitioned in cwy.cu.

usage: python tools/probe_backsweep_scan.py [cfg]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from paper_1209_1910_b200 import workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
d, e, w = W.problem(cfg)
n = len(d)
tn = O.tnorm(d, e)
wt = O.shifts(w, O.clusters(w, tn))


def back_serial(t, b, c):
    x = np.zeros(n + 2)
    for i in range(n - 1, -1, -1):
        x[i] = t[i] - b[i] * x[i + 1] - c[i] * x[i + 2]
    return x[:n]


def back_chunked(t, b, c, L):
    chunks = [(a, min(a + L, n)) for a in range(0, n, L)][::-1]
    maps = []
    for a, bb in chunks:
        p1 = p2 = 0.0
        a1, a2, b1, b2 = 1.0, 0.0, 0.0, 1.0
        for i in range(bb - 1, a - 1, -1):
            pi = t[i] - b[i] * p1 - c[i] * p2
            ai = -b[i] * a1 - c[i] * a2
            bi = -b[i] * b1 - c[i] * b2
            p2, p1, a2, a1, b2, b1 = p1, pi, a1, ai, b1, bi
        maps.append((np.array([[a1, b1], [a2, b2]]), np.array([p1, p2])))
    x = np.zeros(n + 2)
    S = np.zeros(2)
    with np.errstate(all="ignore"):
        for (a, bb), (M, v) in zip(chunks, maps):
            x1, x2 = S
            for i in range(bb - 1, a - 1, -1):
                xi = t[i] - b[i] * x1 - c[i] * x2
                x[i] = xi
                x2, x1 = x1, xi
            S = M @ S + v
    return x[:n]


rng = np.random.default_rng(1)
for j in np.linspace(0, n - 1, 8).astype(int):
    f = O.lu_factor(d, e, wt[j], tn)
    bvec = rng.uniform(-1, 1, n)
    l, piv = f["l"], f["piv"]
    cc = bvec[0]
    y = np.zeros(n)
    for i in range(n - 1):
        bn = bvec[i + 1]
        if piv[i]:
            y[i] = bn
            cc = cc - l[i] * bn
        else:
            y[i] = cc
            cc = bn - l[i] * cc
    y[n - 1] = cc
    u0 = f["u0"]
    u1 = np.r_[f["u1"], 0, 0][:n]
    u2 = np.r_[f["u2"], 0, 0, 0][:n]
    xs = back_serial(y / u0, u1 / u0, u2 / u0)
    errs = []
    for L in (2, 8, 32):
        xc = back_chunked(y / u0, u1 / u0, u2 / u0, L)
        with np.errstate(all="ignore"):
            errs.append(np.abs(xc - xs).max() / np.abs(xs).max())
    print(f"vector {j:5d}: chunked/serial relative error  L=2 {errs[0]:.1e}  L=8 {errs[1]:.1e}  L=32 {errs[2]:.1e}")
