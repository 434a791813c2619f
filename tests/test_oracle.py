"""Pins of the CPU oracle (oracle/) against what the paper and mathematics fix.

Every test compares the oracle with something other than itself: the paper's/SPEC's
hand examples, closed forms, brute force (dense Jacobi, dense products), published
test vectors, or a library routine (numpy QR / eigh, scipy LAPACK).
"Oracle pins" for which test pins which oracle function.
"""
import os

import numpy as np
import pytest

import oracle as O
from paper_1209_1910_b200 import workloads as W
from tests.helpers import (EPS, dense, jacobi_eigh, orth_units, parity_report, residual_units,
                           residual_units_tridiag, sigma_min, vec_diff_upto_sign)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ------------------------------------------------------------------ R1 / R2 / R3

def test_tnorm_spec_examples():
    # SPEC.md:51-53
    assert O.tnorm([5.0], None) == 5.0
    assert O.tnorm([1.0, 1.0, 1.0], [1.0, 1.0]) == 3.0
    assert O.tnorm([10.0, 9.0], [1.0]) == 11.0
    # SPEC.md:84 invariants: >= max|d|, invariant under sign flip of e
    rng = np.random.default_rng(3)
    d, e = rng.normal(size=30), rng.normal(size=29)
    assert O.tnorm(d, e) == O.tnorm(d, -e) >= np.abs(d).max()
    assert O.tnorm(d, e) == pytest.approx(np.abs(dense(d, e)).sum(axis=0).max(), rel=0, abs=1e-15)


def test_cluster_rule_hand():
    # gap 5e-4 <= 1e-3 chains, gap 1 does not
    assert list(O.clusters([1.0, 1.0005], 1.0)) == [0, 2]
    assert list(O.clusters([1.0, 2.0], 1.0)) == [0, 1, 2]
    # equality chains (reading 2: "<=" of Alg. 1/4)
    assert list(O.clusters([0.0, 0.5, 1.5], 1000.0)) == [0, 3]


def test_cluster_rule_laplacian_closed_form():
    # cfg1: lambda_k = 2 - 2cos(k pi/(n+1)); consecutive gap
    # 4 sin((2k+1)pi/(2(n+1))) sin(pi/(2(n+1))) <= 1e-3*||T||_1 = 4e-3 only at the edges.
    n = 200
    k = np.arange(1, n + 1)
    lam = 2.0 - 2.0 * np.cos(k * np.pi / (n + 1))
    gap = 4.0 * np.sin((2 * k[:-1] + 1) * np.pi / (2 * (n + 1))) * np.sin(np.pi / (2 * (n + 1)))
    starts_expected = [0] + [j for j in range(1, n) if gap[j - 1] > 4e-3] + [n]
    cs = O.clusters(lam, 4.0)
    assert list(cs) == starts_expected
    sizes = np.diff(cs)
    # two clusters of 8 at the spectrum edges, 184 singletons
    assert sizes[0] == 8 and sizes[-1] == 8 and (sizes == 1).sum() == 184


def test_cluster_rule_glued_wilkinson():
    # SURVEY Appendix B (erratum of PAPER.md:832 / SPEC.md:400): W21+ glued with small
    # delta forms 14 clusters, 7 of nb and 7 of 2nb, under the 1e-3||T|| rule.
    nb = 5
    d, e = W.glued_wilkinson(nb, 1e-4)
    w = np.linalg.eigvalsh(dense(d, e))          # library eigenvalues, not the oracle's
    cs = O.clusters(w, O.tnorm(d, e))
    sizes = sorted(np.diff(cs).tolist())
    assert sizes == [nb] * 7 + [2 * nb] * 7


def test_shift_ladder_hand():
    u = 2.0 ** -52
    cs = O.clusters([1.0, 1.0], 1.0)
    assert list(O.shifts([1.0, 1.0], cs)) == [1.0, 1.0 + 5 * u]      # 10*eps*|1| = 5 ulp(1)
    cs = O.clusters([1.0, 1.0, 1.0], 1.0)
    assert list(O.shifts([1.0, 1.0, 1.0], cs)) == [1.0, 1.0 + 5 * u, 1.0 + 10 * u]
    w = [0.0, 1.0, 1.0 + 1e-3]                                         # separated: untouched
    cs = O.clusters(w, 1e-4)
    assert list(O.shifts(w, cs)) == w


def test_shift_ladder_strict_inside_clusters():
    d, e, w = W.problem("cfg3", 420)
    tn = O.tnorm(d, e)
    cs = O.clusters(w, tn)
    wt = O.shifts(w, cs)
    assert (wt >= w).all()
    for a, b in zip(cs[:-1], cs[1:]):
        assert (np.diff(wt[a:b]) > 0).all()
        assert wt[a] == w[a]
    assert np.abs(wt - w).max() <= 10 * EPS * np.abs(w).max() * np.diff(cs).max()


# ------------------------------------------------------------------ RNG

def test_splitmix64_golden():
    rows = [l.split() for l in open(os.path.join(GOLDEN, "splitmix64.txt")) if l.strip() and not l.startswith("#")]
    for seed, k, out in rows:
        assert O.splitmix64(int(seed), int(k)) == int(out)


def test_start_vector_range_and_independence():
    b = O.start_vector(1000, 1, 7)
    assert (b >= -1).all() and (b < 1).all()
    assert abs(b.mean()) < 0.1 and abs(b.var() - 1 / 3) < 0.05
    assert not np.array_equal(b, O.start_vector(1000, 1, 8))
    assert not np.array_equal(b, O.start_vector(1000, 1, 7, restart=1))
    assert not np.array_equal(b, O.start_vector(1000, 2, 7))


def test_start_vector_golden_table():
    """Reading 7's (seed, n, j, restart, i) -> value mapping, including the counter layout and
    the top-53-bit conversion, against the table written by tests/golden/make_start_vectors.py
    (plain Python integers, independent of oracle.c)."""
    rows = [l.split() for l in open(os.path.join(GOLDEN, "start_vectors.txt")) if l.strip() and not l.startswith("#")]
    assert len(rows) >= 30
    for seed, n, j, r, i, v in rows:
        b = O.start_vector(int(n), int(seed), int(j), restart=int(r))
        assert b[int(i)] == float.fromhex(v), (seed, n, j, r, i)


# ------------------------------------------------------------------ LU (Eq. 1 solver)

def test_lu_spec_examples():
    f = O.lu_factor([2.0, 2.0], [0.0], 0.0)
    assert list(f["u0"]) == [2.0, 2.0] and f["piv"][0] == 0
    assert list(O.lu_solve(f, [2.0, 4.0])) == [1.0, 2.0]
    f = O.lu_factor([0.0, 0.0], [1.0], 0.0)            # |1| > |0| swaps
    assert f["piv"][0] == 1


@pytest.mark.parametrize("n", [1, 2, 3, 6, 17, 50])
def test_lu_vs_dense_solve(n):
    rng = np.random.default_rng(n)
    d, e = rng.uniform(-1, 1, n), rng.uniform(-1, 1, max(n - 1, 0))
    shift = 0.3
    b = rng.normal(size=n)
    x = O.lu_solve(O.lu_factor(d, e, shift), b)
    A = dense(d, e) - shift * np.eye(n)
    xr = np.linalg.solve(A, b)
    # relative residual <= c n eps, c ~ 100
    assert np.abs(A @ x - b).max() <= 100 * n * EPS * (np.abs(A).sum(axis=0).max() * np.abs(x).max() + np.abs(b).max())
    assert np.abs(x - xr).max() <= 1e-10 * np.abs(xr).max()


def test_lu_singular_shift_finite_and_floor():
    # T = [[1,1],[1,1]] is singular at shift 0: the pivot floor keeps the solve finite
    # and the solution points along the null vector [1,-1]/sqrt(2).
    f = O.lu_factor([1.0, 1.0], [1.0], 0.0)
    assert abs(f["u0"][1]) == EPS * 2.0                   # floored to eps*||T||_1
    x = O.lu_solve(f, [1.0, 0.3])
    assert np.isfinite(x).all()
    v = x / np.linalg.norm(x)
    assert vec_diff_upto_sign(v, np.array([1.0, -1.0]) / np.sqrt(2)) < 1e-14
    # zero pivot takes the + sign
    f = O.lu_factor([0.0, 1.0], [0.0], 0.0)
    assert f["u0"][0] == EPS * 1.0


# ------------------------------------------------------------------ reflector (Eq. 2)

def test_reflector_spec_examples():
    y, c, t, _ = O.reflector([1.0, 0.0, 0.0])
    assert c == -1.0 and list(y) == [2.0, 0.0, 0.0] and t == 0.5
    y, c, t, _ = O.reflector([0.0, 5.0])               # SPEC.md:197, sgn(0)=+1
    assert c == -5.0 and list(y) == [5.0, 5.0] and t == pytest.approx(0.04, rel=1e-15)


def test_reflector_identities():
    rng = np.random.default_rng(5)
    for _ in range(200):
        m = rng.integers(1, 12)
        u = rng.normal(size=m) * 10.0 ** rng.uniform(-5, 5)
        y, c, t, _ = O.reflector(u)
        H = np.eye(m) - t * np.outer(y, y)
        e1 = np.zeros(m)
        e1[0] = 1.0
        assert np.abs(H @ u - c * e1).max() <= 1e-13 * np.linalg.norm(u)   # H u = c e_1
        assert abs(t * (y @ y) - 2.0) <= 1e-14 * 4                          # t = 2/||y||^2
        assert np.abs(H @ H.T - np.eye(m)).max() <= 1e-14 * 8


# ------------------------------------------------------------------ compact WY (Eqs. 3-4, §3.3)

def _dense_householder_product(Y, T):
    n, m = Y.shape
    P = np.eye(n)
    for k in range(m):
        P = P @ (np.eye(n) - T[k, k] * np.outer(Y[:, k], Y[:, k]))
    return P


def test_eq4_compact_wy_identity():
    # SPEC.md:494 acceptance 1: I - Y T Y^T == H_1 ... H_m entrywise <= 1e-13
    rng = np.random.default_rng(11)
    for _ in range(60):
        n = int(rng.integers(1, 21))
        m = int(rng.integers(1, n + 1))
        V = rng.normal(size=(n, m))
        Y, T = O.cwy_build(V)
        assert np.allclose(np.tril(Y), Y) and np.allclose(np.triu(T), T)
        for k in range(m):
            assert abs(T[k, k] * (Y[:, k] @ Y[:, k]) - 2.0) <= 1e-13     # t_k = 2/||y_k||^2
        lhs = np.eye(n) - Y @ T @ Y.T
        assert np.abs(lhs - _dense_householder_product(Y, T)).max() <= 1e-13


def test_cwy_apply_block_is_householder_q():
    """Blocked look-ahead oracle: U = (I - Y T Y^T)^T X with Y, T from k
    columns of V is Q^T X for the complete Q of LAPACK's Householder QR of V (dgeqrf/dorgqr:
    H_1 .. H_k with the same sign convention beta = -sign(alpha) ||.||), and the untransposed
    application is Q X.  Independent of the oracle's own Y/T algebra."""
    rng = np.random.default_rng(14)
    for n, k, b in [(6, 1, 1), (12, 5, 3), (40, 17, 8), (120, 60, 8)]:
        V = rng.normal(size=(n, k))
        X = rng.normal(size=(n, b))
        Q, _ = np.linalg.qr(V, mode="complete")
        assert np.abs(O.cwy_apply_block(V, X, trans=True) - Q.T @ X).max() <= 1e-12 * max(1.0, np.abs(X).max())
        assert np.abs(O.cwy_apply_block(V, X, trans=False) - Q @ X).max() <= 1e-12 * max(1.0, np.abs(X).max())
    # k = 0: nothing applied
    X = rng.normal(size=(9, 2))
    assert np.array_equal(O.cwy_apply_block(np.zeros((9, 0)), X), X)


def test_cwy_equals_householder_qr():
    # Householder-QR special case: cWY-orthogonalising V yields QR(V)'s Q up to column signs.
    rng = np.random.default_rng(12)
    for n, m in [(5, 1), (8, 8), (30, 12), (200, 50)]:
        V = rng.normal(size=(n, m))
        Qr, _ = np.linalg.qr(V)
        for Q in (O.cwy_orth(V), O.cwy_ordinary_orth(V), O.householder_orth(V)):
            for k in range(m):
                assert vec_diff_upto_sign(Q[:, k], Qr[:, k]) <= 1e-12


def test_cwy_variants_agree_and_flip_sign():
    rng = np.random.default_rng(13)
    V = rng.normal(size=(40, 15))
    Qp = O.cwy_orth(V)              # §3.3.2: q = (Y T Y^T - I) e_j
    Qo = O.cwy_ordinary_orth(V)     # §3.3.1: q = (I - Y T Y^T) e_j
    Qh = O.householder_orth(V)      # Alg. 2
    assert np.abs(Qp + Qo).max() <= 1e-13       # exactly the flipped sign
    assert np.abs(Qo - Qh).max() <= 1e-13


def test_cwy_orthogonality_independent_of_condition():
    # Table 1: O(eps) for Householder / cWY vs O(eps kappa) for MGS.
    rng = np.random.default_rng(14)
    n, m = 200, 50
    Q0, _ = np.linalg.qr(rng.normal(size=(n, m)))
    R, _ = np.linalg.qr(rng.normal(size=(m, m)))
    for kappa in (1e2, 1e4, 1e6, 1e8):
        s = np.logspace(0, -np.log10(kappa), m)
        V = Q0 @ np.diag(s) @ R
        Q = O.cwy_orth(V)
        assert np.abs(Q.T @ Q - np.eye(m)).max() <= 100 * n * EPS
    # MGS on the kappa=1e8 matrix loses orthogonality (test-side MGS, contrast only)
    Qm = V.copy()
    for j in range(m):
        for i in range(j):
            Qm[:, j] -= (Qm[:, i] @ Qm[:, j]) * Qm[:, i]
        Qm[:, j] /= np.linalg.norm(Qm[:, j])
    assert np.abs(Qm.T @ Qm - np.eye(m)).max() > 1e3 * np.abs(Q.T @ Q - np.eye(m)).max()


# ------------------------------------------------------------------ bisection (R5)

def test_sturm_spec_examples():
    assert O.sturm_count([0.0], None, 1.0) == 1
    assert O.sturm_count([0.0], None, -1.0) == 0
    # SPEC.md:127 (eigenvalues 1-sqrt2, 1, 1+sqrt2): one eigenvalue below 1.  x = 1 itself
    # is an eigenvalue; the zero-pivot convention of SPEC.md:144 / LAPACK (-pivmin) counts
    # it as below (reading R5), so the example is checked just off the point.
    assert O.sturm_count([1.0, 1.0, 1.0], [1.0, 1.0], 1.0 - 1e-12) == 1
    assert O.sturm_count([1.0, 1.0, 1.0], [1.0, 1.0], 1.0 + 1e-12) == 2
    assert O.sturm_count([1.0, 1.0, 1.0], [1.0, 1.0], 1.0) == 2


def test_sturm_monotone_and_endpoints():
    d, e = W.random_sym(300, 4)
    xs = np.linspace(-4, 4, 401)
    cnt = [O.sturm_count(d, e, x) for x in xs]
    assert cnt[0] == 0 and cnt[-1] == 300 and all(a <= b for a, b in zip(cnt, cnt[1:]))


def test_bisect_laplacian_closed_form():
    n = 200
    d, e = W.laplacian(n)
    w = O.bisect(d, e)
    k = np.arange(1, n + 1)
    lam = 2.0 - 2.0 * np.cos(k * np.pi / (n + 1))
    assert np.abs(w - lam).max() <= 10 * EPS * 4.0


def test_bisect_all_ones_closed_form():
    n = 100
    d, e = W.all_ones(n)
    w = O.bisect(d, e)
    k = np.arange(n, 0, -1)
    lam = 1.0 + 2.0 * np.cos(k * np.pi / (n + 1))       # SPEC.md:135, ascending
    assert np.abs(w - lam).max() <= 10 * EPS * 3.0


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8])
def test_bisect_vs_jacobi(n):
    rng = np.random.default_rng(100 + n)
    d, e = rng.normal(size=n), rng.normal(size=n - 1)
    wj, _ = jacobi_eigh(dense(d, e))
    assert np.abs(O.bisect(d, e) - wj).max() <= 1e-13 * max(1.0, np.abs(wj).max())


def test_bisect_vs_lapack():
    # LAPACK DSTEBZ (the paper's eigenvalue routine) as library cross-check
    d, e = W.random_sym(2000, 0)
    w = O.bisect(d, e)
    assert np.abs(w - W.eigenvalues(d, e, "stebz")).max() <= 20 * EPS * O.tnorm(d, e)


# ------------------------------------------------------------------ Alg. 4 end to end

def test_eigvecs_trivial_cases():
    Z, info = O.eigvecs([3.0], None, [3.0])
    assert info == 0 and Z.shape == (1, 1) and Z[0, 0] == 1.0
    Z, info = O.eigvecs(np.zeros(4), np.zeros(3), np.zeros(4))      # ||T||_1 = 0 -> I
    assert info == 0 and np.array_equal(Z, np.eye(4))


def test_eigvecs_diagonal_matrix():
    d = np.array([3.0, -1.0, 2.0, 7.0, 0.5])
    w = np.sort(d)
    Z, info = O.eigvecs(d, np.zeros(4), w)
    assert info == 0
    order = np.argsort(d)
    assert np.abs(Z - np.eye(5)[:, order]).max() <= 1e-14


def _laplacian_vectors(n):
    i = np.arange(1, n + 1)[:, None]
    k = np.arange(1, n + 1)[None, :]
    return np.sqrt(2.0 / (n + 1)) * np.sin(i * k * np.pi / (n + 1))


def test_eigvecs_laplacian_closed_form():
    # cfg1 (BASELINE configs[0]): v_jk = sqrt(2/(n+1)) sin(jk pi/(n+1)).
    n = 200
    d, e = W.laplacian(n)
    k = np.arange(1, n + 1)
    lam = 2.0 - 2.0 * np.cos(k * np.pi / (n + 1))
    Z, info, its = O.eigvecs(d, e, lam, seed=1, return_iters=True)
    assert info == 0 and (its == 2).all()
    V = _laplacian_vectors(n)
    cs = O.clusters(lam, 4.0)
    for a, b in zip(cs[:-1], cs[1:]):
        if b - a == 1:
            assert vec_diff_upto_sign(Z[:, a], V[:, a]) <= 1e-10
        else:
            assert sigma_min(Z[:, a:b], V[:, a:b]) >= 1 - 1e-10
    assert residual_units(d, e, lam, Z) <= 10 and orth_units(Z) <= 10


def test_eigvecs_all_ones_closed_form():
    n = 100
    d, e = W.all_ones(n)
    k = np.arange(n, 0, -1)
    lam = 1.0 + 2.0 * np.cos(k * np.pi / (n + 1))
    Z, info = O.eigvecs(d, e, lam, seed=3)
    assert info == 0
    i = np.arange(1, n + 1)[:, None]
    V = np.sqrt(2.0 / (n + 1)) * np.sin(i * k[None, :] * np.pi / (n + 1))
    wr, vr, nv, ng = parity_report(lam, 3.0, Z, V, tau_rel=1e-3)
    assert wr <= 1e-10 and vr >= 1 - 1e-10
    assert residual_units(d, e, lam, Z) <= 10 and orth_units(Z) <= 10


@pytest.mark.parametrize("n", [2, 3, 5, 8])
def test_eigvecs_vs_jacobi(n):
    rng = np.random.default_rng(200 + n)
    d, e = rng.normal(size=n), rng.normal(size=n - 1)
    wj, Vj = jacobi_eigh(dense(d, e))
    Z, info = O.eigvecs(d, e, wj, seed=5)
    assert info == 0
    for k in range(n):
        assert vec_diff_upto_sign(Z[:, k], Vj[:, k]) <= 1e-10


def test_eigvecs_glued_wilkinson_type3():
    # SPEC.md:500 acceptance 7 (corrected cluster count): n = 105, delta = 1e-4
    d, e = W.glued_wilkinson(5, 1e-4)
    w = W.eigenvalues(d, e)
    Z, info, its = O.eigvecs(d, e, w, seed=1, return_iters=True)
    assert info == 0 and (its <= 5).all()
    assert residual_units(d, e, w, Z) <= 10 and orth_units(Z) <= 10
    _, V = np.linalg.eigh(dense(d, e))
    tn = O.tnorm(d, e)
    cs = O.clusters(w, tn)
    for a, b in zip(cs[:-1], cs[1:]):
        assert sigma_min(Z[:, a:b], V[:, a:b]) >= 1 - 1e-10


def test_eigvecs_cfg2_vs_lapack():
    # cfg2 (configs[1]) in full: invariants + P3 parity against LAPACK's eigenvectors.
    import scipy.linalg as sl

    d, e, w = W.problem("cfg2")
    Z, info, its = O.eigvecs(d, e, w, seed=1, return_iters=True)
    assert info == 0 and its.max() <= 5
    assert residual_units_tridiag(d, e, w, Z) <= 10 and orth_units(Z) <= 10
    _, V = sl.eigh_tridiagonal(d, e)
    worst_vec, worst_sig, nv, ng = parity_report(w, O.tnorm(d, e), Z, V)
    assert nv > 1900 and worst_vec <= 1e-10 and worst_sig >= 1 - 1e-10


@pytest.mark.parametrize("cfg,n", [("cfg3", 1050), ("cfg4", 300), ("cfg5", 600), ("type1", 1050),
                                   ("type2", 300), ("type3", 420)])
def test_eigvecs_invariants_scaled_configs(cfg, n):
    d, e, w = W.problem(cfg, n)
    Z, info = O.eigvecs(d, e, w, seed=1)
    assert info == 0
    assert residual_units_tridiag(d, e, w, Z) <= 10
    assert orth_units(Z) <= 10


def test_eigvecs_deterministic_and_range_consistent():
    d, e, w = W.problem("cfg3", 420)
    Z1, _ = O.eigvecs(d, e, w, seed=1)
    Z2, _ = O.eigvecs(d, e, w, seed=1)
    assert np.array_equal(Z1, Z2)
    Zr, _ = O.eigvecs(d, e, w, seed=1, j_lo=50, j_hi=130)
    assert np.array_equal(Zr, Z1[:, 50:130])


def test_eigvecs_seed_insensitive_where_determined():
    # Reading 7: different start vectors give the same determined vectors.
    d, e, w = W.problem("cfg2", 600)
    Z1, _ = O.eigvecs(d, e, w, seed=1)
    Z2, _ = O.eigvecs(d, e, w, seed=2)
    worst_vec, worst_sig, nv, ng = parity_report(w, O.tnorm(d, e), Z1, Z2)
    assert worst_vec <= 1e-10 and worst_sig >= 1 - 1e-10


# ---------------------------------------------------------------- Alg. 1 (classical MGS)
# the comparison path.  Pinned by the closed-form Laplacian vectors, by
# LAPACK on cfg2, by the glued-Wilkinson subspaces, and by the compact-WY oracle (the two
# reorthogonalisations orthogonalise the same solve outputs; they agree up to rounding where
# the vectors are determined).


def test_eigvecs_mgs_laplacian_closed_form():
    n = 200
    d, e = W.laplacian(n)
    k = np.arange(1, n + 1)
    lam = 2.0 - 2.0 * np.cos(k * np.pi / (n + 1))
    Z, info, its = O.eigvecs(d, e, lam, seed=1, return_iters=True, mgs=True)
    assert info == 0 and (its == 2).all()
    V = _laplacian_vectors(n)
    cs = O.clusters(lam, 4.0)
    for a, b in zip(cs[:-1], cs[1:]):
        if b - a == 1:
            assert vec_diff_upto_sign(Z[:, a], V[:, a]) <= 1e-10
        else:
            assert sigma_min(Z[:, a:b], V[:, a:b]) >= 1 - 1e-10
    assert residual_units(d, e, lam, Z) <= 10 and orth_units(Z) <= 10


def test_eigvecs_mgs_cfg2_vs_lapack_and_cwy():
    import scipy.linalg as sl

    d, e, w = W.problem("cfg2", 1200)
    Z, info = O.eigvecs(d, e, w, seed=1, mgs=True)
    assert info == 0
    assert residual_units_tridiag(d, e, w, Z) <= 10 and orth_units(Z) <= 10
    _, V = sl.eigh_tridiagonal(d, e)
    worst_vec, worst_sig, nv, ng = parity_report(w, O.tnorm(d, e), Z, V)
    assert nv > 1100 and worst_vec <= 1e-10 and worst_sig >= 1 - 1e-10
    Zc, _ = O.eigvecs(d, e, w, seed=1)
    assert np.abs(Z - Zc).max() <= 1e-12       # same solves, same sign rule


def test_eigvecs_mgs_glued_wilkinson_subspaces():
    d, e = W.glued_wilkinson(5, 1e-4)
    w = W.eigenvalues(d, e)
    Z, info = O.eigvecs(d, e, w, seed=1, mgs=True)
    assert info == 0
    assert residual_units(d, e, w, Z) <= 10 and orth_units(Z) <= 10
    _, V = np.linalg.eigh(dense(d, e))
    cs = O.clusters(w, O.tnorm(d, e))
    for a, b in zip(cs[:-1], cs[1:]):
        assert sigma_min(Z[:, a:b], V[:, a:b]) >= 1 - 1e-10


@pytest.mark.parametrize("cfg,n", [("cfg3", 630), ("type3", 420)])
def test_eigvecs_mgs_invariants_and_range(cfg, n):
    d, e, w = W.problem(cfg, n)
    Z, info = O.eigvecs(d, e, w, seed=1, mgs=True)
    assert info == 0
    assert residual_units_tridiag(d, e, w, Z) <= 10 and orth_units(Z) <= 10
    Zr, _ = O.eigvecs(d, e, w, seed=1, j_lo=40, j_hi=110, mgs=True)
    assert np.array_equal(Zr, Z[:, 40:110])


# ------------------------------------------------------------------ silent branches (readings 9, 16, 17)

def test_restart_branch_closed_form():
    """Reading 16 (PAPER.md:681-716 is silent on an iterate inside the accepted span): with
    T = diag(1, 2) and the (wrong) input w = [1, 1], both shifts sit on eigenvalue 1 and form
    one cluster.  The second vector's first iterate lies in span(e_1) = span(z_1) up to
    rounding, so ||uhat|| <= n eps ||x|| triggers a restart; the restarted iterate is
    reorthogonalised to the complement.  Closed form: z_0 = e_1, z_1 = e_2 (the only unit
    vectors orthogonal to each other with z_0 the eigenvector for shift 1); the restart
    shows in the iteration count (> 2 = one restart plus 2 passes)."""
    Z, info, its = O.eigvecs(np.array([1.0, 2.0]), np.array([0.0]), np.array([1.0, 1.0]), seed=1,
                             return_iters=True)
    assert info == 0
    assert np.abs(Z - np.eye(2)).max() <= 1e-15
    assert its[0] == 2 and its[1] > 2, its


def test_maxits_flag_closed_form():
    """Readings 9 and 17: a vector that never passes the growth test in MAXITS = 5 iterations is
    kept and counted in the return value.  T = 1e-20 diag(1, 3, 5, 5.002, 5.004) with shifts at
    distance >= 0.5e-20 from every eigenvalue (a singleton and a 1e-3 ||T||_1 cluster of 3 +
    one more singleton): for a diagonal T the solve is x_i = sigma b_i / (d_i - w), and
    sigma = n ||T||_1 max(eps, |u_nn|) / ||b||_1 = n ||T||_1 eps / ||b||_1 since |u_nn| < eps,
    so ||x||_inf <= n ||T||_1 eps / 0.5e-20 = 5 * 5.004 * 2 eps < sqrt(0.1 / n) on every
    iteration (the cWY iterate c q has norm <= ||x||): no vector ever counts a pass."""
    s = 1e-20
    d = s * np.array([1.0, 3.0, 5.0, 5.002, 5.004])
    e = np.zeros(4)
    w = s * np.array([2.0, 3.6, 6.0, 6.0 + 1e-6, 6.0 + 2e-6])
    cs = O.clusters(w, O.tnorm(d, e))
    assert list(cs) == [0, 1, 2, 5]                    # singleton, singleton, cluster of 3
    Z, info, its = O.eigvecs(d, e, w, seed=1, return_iters=True)
    assert info == 5, info
    assert (its == 5).all(), its                      # MAXITS, no restart
    assert np.isfinite(Z).all()
    assert np.allclose(np.linalg.norm(Z, axis=0), 1.0, atol=1e-14)


def test_rescaling_reading21_scale_free():
    """Reading 21: outside ||T||_1 in [2^-200, 2^200] the oracle works on 2^k T (||2^k T||_1 in
    [1, 2)), so 2^300 T, 2^-500 T and 2^-1000 T (all outside the window) reduce to the SAME
    scaled matrix and give bit-identical vectors; inside the window (2^150 T) nothing is
    rescaled.  All of them are eigenvectors of the unscaled T (P0) and agree with the unscaled
    run within the parity tolerances (P1-P3)."""
    d, e, w = W.problem("cfg2", 300)
    Z0, _ = O.eigvecs(d, e, w, seed=1)
    outs = {}
    for k in (300, -500, -1000, 150):
        s = 2.0 ** k
        Z, info = O.eigvecs(d * s, e * s, w * s, seed=1)
        assert info == 0
        assert residual_units(d, e, w, Z) <= 10 and orth_units(Z) <= 10
        wv, ws, _, _ = parity_report(w, O.tnorm(d, e), Z, Z0)
        assert wv <= 1e-10 and ws >= 1 - 1e-10
        outs[k] = Z
    assert np.array_equal(outs[300], outs[-500]) and np.array_equal(outs[300], outs[-1000])


def test_cfg5_golden_columns_are_eigenvectors():
    """tests/golden/cfg5_oracle_cols.npz (written by tests/golden/make_cfg5_golden.py from a
    full oracle run on cfg5, n = 16000, one cluster): the stored columns are unit eigenvectors
    of T for the stored w (residual <= 10 n eps ||T||_1, the P0 bound), mutually orthogonal,
    the stored w is the workload's (hash and values), and every vector took 2 iterations."""
    import hashlib

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cfg5_oracle_cols.npz")
    if not os.path.exists(path):
        pytest.skip("cfg5 golden columns not generated")
    g = np.load(path)
    d, e, w = W.problem("cfg5")
    n = len(d)
    wg = np.asarray(g["w"])
    assert g["w_sha"].item().decode() == hashlib.sha256(np.ascontiguousarray(wg).tobytes()).hexdigest()
    tn = O.tnorm(d, e)
    assert np.abs(wg - w).max() <= 1e3 * EPS * tn
    assert int(g["info"]) == 0 and (np.asarray(g["iters"]) == 2).all()
    cols = np.asarray(g["cols"])
    Z = np.asarray(g["Z"])
    TZ = d[:, None] * Z
    TZ[:-1] += e[:, None] * Z[1:]
    TZ[1:] += e[:, None] * Z[:-1]
    res = np.linalg.norm(TZ - Z * wg[cols][None, :], axis=0).max() / (n * EPS * tn)
    assert res <= 10.0, res
    G = Z.T @ Z
    assert np.abs(G - np.eye(len(cols))).max() / (n * EPS) <= 10.0
