"""Test-only helpers: brute-force references and the parity metrics of SURVEY §8(c).

Nothing here is used by the product path.  ``jacobi_eigh`` is an independent dense
cyclic-Jacobi eigensolver (brute force for n <= 8 pins)."""
from __future__ import annotations

import numpy as np

EPS = 2.0 ** -53


def dense(d, e):
    d = np.asarray(d, dtype=np.float64)
    T = np.diag(d)
    if d.shape[0] > 1:
        T = T + np.diag(e, 1) + np.diag(e, -1)
    return T


def jacobi_eigh(A, sweeps=100):
    """Cyclic Jacobi rotations until off-diagonal mass is negligible.  Returns ascending
    eigenvalues and the matching orthonormal eigenvectors (columns)."""
    A = np.array(A, dtype=np.float64)
    n = A.shape[0]
    V = np.eye(n)
    for _ in range(sweeps):
        off = np.sqrt(np.sum((A - np.diag(np.diag(A))) ** 2))
        if off < 1e-300 or off <= 1e-17 * np.sqrt(np.sum(A ** 2)):
            break
        for p in range(n - 1):
            for q in range(p + 1, n):
                if abs(A[p, q]) <= 1e-300 or abs(A[p, q]) <= 1e-18 * (abs(A[p, p]) + abs(A[q, q])):
                    A[p, q] = A[q, p] = 0.0
                    continue
                theta = (A[q, q] - A[p, p]) / (2.0 * A[p, q])
                t = np.sign(theta) / (abs(theta) + np.sqrt(theta * theta + 1.0)) if theta != 0 else 1.0
                c = 1.0 / np.sqrt(t * t + 1.0)
                s = t * c
                J = np.eye(n)
                J[p, p] = c
                J[q, q] = c
                J[p, q] = s
                J[q, p] = -s
                A = J.T @ A @ J
                V = V @ J
    w = np.diag(A).copy()
    idx = np.argsort(w, kind="stable")
    return w[idx], V[:, idx]


def residual_units(d, e, w, Z):
    """max_j ||T z_j - w_j z_j||_2 / (n eps ||T||_1)   (P0, BASELINE.json north_star)."""
    T = dense(d, e)
    n = T.shape[0]
    tn = np.abs(T).sum(axis=0).max()
    r = np.linalg.norm(T @ Z - Z * np.asarray(w)[None, :], axis=0).max()
    return r / (n * EPS * tn) if tn > 0 else r


def residual_units_tridiag(d, e, w, Z):
    """Same as residual_units without forming T densely (large n)."""
    d = np.asarray(d)
    n = d.shape[0]
    TZ = d[:, None] * Z
    if n > 1:
        TZ[:-1] += e[:, None] * Z[1:]
        TZ[1:] += e[:, None] * Z[:-1]
    tn = np.abs(d).copy()
    if n > 1:
        tn[:-1] += np.abs(e)
        tn[1:] += np.abs(e)
    tn = tn.max()
    r = np.linalg.norm(TZ - Z * np.asarray(w)[None, :], axis=0).max()
    return r / (n * EPS * tn) if tn > 0 else r


def orth_units(Z):
    """max |Z^T Z - I| / (n eps)   (P0)."""
    n = Z.shape[0]
    G = Z.T @ Z
    return np.abs(G - np.eye(G.shape[0])).max() / (n * EPS)


def sign_fix(Z):
    """Canonical sign: largest-|entry| positive, lowest index on ties (reading 15)."""
    Z = np.array(Z, dtype=np.float64, copy=True)
    idx = np.argmax(np.abs(Z), axis=0)
    s = np.sign(Z[idx, np.arange(Z.shape[1])])
    s[s == 0] = 1.0
    return Z * s[None, :]


def vec_diff_upto_sign(a, b):
    return min(np.abs(a - b).max(), np.abs(a + b).max())


def sigma_min(A, B):
    """Smallest singular value of A^T B (subspace agreement, P2)."""
    return np.linalg.svd(A.T @ B, compute_uv=False).min()


def groups(w, thr):
    """Maximal runs of consecutive w with gaps <= thr, as (start, stop) pairs."""
    n = len(w)
    out = []
    s = 0
    for j in range(1, n + 1):
        if j == n or not (w[j] - w[j - 1] <= thr):
            out.append((s, j))
            s = j
    return out


def parity_report(w, tn, Za, Zb, tau_rel=1e-6):
    """P1-P3 of SURVEY §8(c): per-vector agreement (up to sign) for vectors whose gaps
    to both neighbours exceed tau_rel*||T||_1, subspace agreement (sigma_min) for runs
    chained at that gap.  Returns (max per-vector diff, min sigma, n_vec, n_groups)."""
    worst_vec = 0.0
    worst_sig = 1.0
    nv = ng = 0
    for s, t in groups(w, tau_rel * tn):
        if t - s == 1:
            worst_vec = max(worst_vec, vec_diff_upto_sign(Za[:, s], Zb[:, s]))
            nv += 1
        else:
            worst_sig = min(worst_sig, sigma_min(Za[:, s:t], Zb[:, s:t]))
            ng += 1
    return worst_vec, worst_sig, nv, ng
