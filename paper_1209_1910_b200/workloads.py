"""Seeded synthetic inputs shared by tests, bench.py and smoke() -- no method arithmetic.

Matrix families are the paper's (§5.1) and BASELINE.json's five
configs; every matrix is a formula or a numpy PCG64 draw
(``default_rng(seed)``, d drawn first, then e).  The eigenvalues w are the
path's INPUT (the paper computes them with LAPACK's bisection DSTEBZ before the timed
eigenvector phase); here they come from LAPACK through scipy: DSTEBZ
as in the paper for n <= 4200, DSTEMR above (DSTEBZ takes 78 s at n=16000; the two agree
within ~2e2 eps ||T||_1, far inside the path's tolerances).  Neither the oracle nor the CUDA path is used to make inputs.
"""
from __future__ import annotations

import numpy as np

CONFIGS = ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5")


def laplacian(n: int):
    """cfg1: 1D Laplacian d_i = 2, e_i = -1 (BASELINE.json configs[0])."""
    return np.full(n, 2.0), np.full(n - 1, -1.0)


def random_sym(n: int, seed: int = 0, lo: float = -1.0, hi: float = 1.0):
    """cfg2 (configs[1]): d, e iid uniform(lo, hi); Type 1 of the paper is lo=0, hi=1
    (PAPER.md:780)."""
    rng = np.random.default_rng(seed)
    d = rng.uniform(lo, hi, n)
    e = rng.uniform(lo, hi, n - 1)
    return d, e


def all_ones(n: int):
    """Type 2: all-ones tridiagonal."""
    return np.ones(n), np.ones(n - 1)


def wilkinson21():
    """W21+ (PAPER.md:816-828): d = 10, 9, ..., 1, 0, 1, ..., 10; e = 1."""
    return np.abs(10.0 - np.arange(21, dtype=np.float64)), np.ones(20)


def glued_wilkinson(nblocks: int, delta: float):
    """W_g+ (PAPER.md:798-835): nblocks copies of W21+ glued by delta."""
    d1, e1 = wilkinson21()
    d = np.tile(d1, nblocks)
    e = np.ones(21 * nblocks - 1)
    if nblocks > 1:
        e[20::21] = delta
    return d, e


def giant_cluster(n: int, seed: int = 0):
    """cfg4 (configs[3]): d = 1 + 1e-7 U(0,1), e = 1e-9 U(0,1)."""
    rng = np.random.default_rng(seed)
    d = 1.0 + 1e-7 * rng.uniform(0.0, 1.0, n)
    e = 1e-9 * rng.uniform(0.0, 1.0, n - 1)
    return d, e


def perturbed_laplacian(n: int, seed: int = 0):
    """cfg5 (configs[4]): d = 2 + 1e-6 U(-1,1), e = -1."""
    rng = np.random.default_rng(seed)
    d = 2.0 + 1e-6 * rng.uniform(-1.0, 1.0, n)
    e = np.full(n - 1, -1.0)
    return d, e


def make(cfg: str, n: int | None = None, seed: int = 0):
    """(d, e) of a named config.  ``n`` overrides the size (a scaled copy of the same
    family, used for oracle-sized parity cases)."""
    if cfg == "cfg1":
        return laplacian(n or 200)
    if cfg == "cfg2":
        return random_sym(n or 2000, seed)
    if cfg == "cfg3":
        nb = (n or 4200) // 21
        return glued_wilkinson(nb, 1e-10)
    if cfg == "cfg4":
        return giant_cluster(n or 8000, seed)
    if cfg == "cfg5":
        return perturbed_laplacian(n or 16000, seed)
    if cfg == "type1":
        return random_sym(n or 1050, seed, 0.0, 1.0)
    if cfg == "type2":
        return all_ones(n or 1050)
    if cfg == "type3":
        return glued_wilkinson((n or 1050) // 21, 1e-4)
    raise ValueError(f"unknown config {cfg!r}")


STEBZ_MAX_N = 4200


def eigenvalues(d, e, driver: str | None = None):
    """Ascending eigenvalues of T (the path's input w) from LAPACK via scipy."""
    import scipy.linalg as sl

    d = np.asarray(d, dtype=np.float64)
    if d.shape[0] == 1:
        return d.copy()
    if driver is None:
        driver = "stebz" if d.shape[0] <= STEBZ_MAX_N else "stemr"
    return sl.eigvalsh_tridiagonal(d, np.asarray(e, dtype=np.float64), lapack_driver=driver)


def problem(cfg: str, n: int | None = None, seed: int = 0):
    d, e = make(cfg, n, seed)
    return d, e, eigenvalues(d, e)
