"""GPU parity: the C-ABI product path (libtinv.so via paper_1209_1910_b200.tinv) against
the CPU oracle on the same seeded inputs.

Contract (BASELINE.json north_star):
  P0  max_j ||T z_j - w_j z_j||_2 <= 10 n eps ||T||_1 and max|Z^T Z - I| <= 10 n eps
  P1/P3  vectors whose gaps to both neighbours exceed 1e-6 ||T||_1 agree with the oracle
      up to sign within 1e-10 (max-norm); P2/P3 runs chained at that gap agree as
      subspaces: sigma_min(Z_gpu^T Z_oracle) >= 1 - 1e-10.
Full-size configs the oracle cannot finish in seconds (cfg4, cfg5) are checked with the
invariants at full size plus sampled columns the oracle computes (its range mode).
"""
import hashlib
import os

import numpy as np
import pytest

import oracle as O
from paper_1209_1910_b200 import workloads as W
from tests.helpers import EPS, groups, parity_report, sigma_min, vec_diff_upto_sign

pytestmark = pytest.mark.gpu

TOL_VEC = 1e-10
TOL_SUB = 1e-10


@pytest.fixture(scope="module")
def torch():
    import torch as t

    assert t.cuda.is_available()
    return t


@pytest.fixture(scope="module")
def handle(torch):
    from paper_1209_1910_b200.tinv import Tinv

    h = Tinv(0)
    yield h
    h.close()


def run_gpu(handle, torch, d, e, w, seed=1):
    dev = torch.device("cuda:0")
    dt = torch.tensor(d, dtype=torch.float64, device=dev)
    et = torch.tensor(e if len(d) > 1 else np.zeros(1), dtype=torch.float64, device=dev)
    wt = torch.tensor(w, dtype=torch.float64, device=dev)
    Z, rc = handle.eigvecs(dt, et, wt, seed=seed)
    torch.cuda.synchronize()
    return Z, rc


def invariants_gpu(torch, d, e, w, Z):
    """P0 on the device (fp64 cuBLAS for Z^T Z; elementwise residual)."""
    n = len(d)
    dev = Z.device
    dt = torch.tensor(d, dtype=torch.float64, device=dev)
    wt = torch.tensor(w, dtype=torch.float64, device=dev)
    TZ = dt[:, None] * Z
    if n > 1:
        et = torch.tensor(e, dtype=torch.float64, device=dev)
        TZ[:-1] += et[:, None] * Z[1:]
        TZ[1:] += et[:, None] * Z[:-1]
    tn = O.tnorm(d, e)
    res = torch.linalg.vector_norm(TZ - Z * wt[None, :], dim=0).max().item() / (n * EPS * tn)
    G = Z.t() @ Z
    G.diagonal().sub_(1.0)
    orth = G.abs().max().item() / (n * EPS)
    return res, orth


def full_parity(handle, torch, d, e, w, seed=1):
    Zg, rc = run_gpu(handle, torch, d, e, w, seed)
    assert rc == 0, f"tinv_eigvecs returned {rc}"
    res, orth = invariants_gpu(torch, d, e, w, Zg)
    assert res <= 10.0, f"residual {res} x n eps ||T||"
    assert orth <= 10.0, f"orthogonality {orth} x n eps"
    Zo, info = O.eigvecs(d, e, w, seed=seed)
    assert info == 0
    Zg_h = Zg.cpu().numpy()
    wv, ws, nv, ng = parity_report(w, O.tnorm(d, e), Zg_h, Zo)
    assert wv <= TOL_VEC, f"per-vector diff {wv}"
    assert ws >= 1 - TOL_SUB, f"subspace sigma_min {ws}"
    return Zg_h, Zo, (res, orth, wv, ws, nv, ng)


# ------------------------------------------------------------------ BASELINE configs

def test_cfg1_laplacian_full(handle, torch):
    d, e, w = W.problem("cfg1")
    Zg, Zo, rep = full_parity(handle, torch, d, e, w)
    # the canonical sign rule (reading 15) makes determined vectors identical wherever the
    # largest |entry| is unique beyond rounding (the Laplacian's symmetric vectors have two
    # mirror-image maxima, where the rule is decided by rounding and only +-z is defined)
    tn = O.tnorm(d, e)
    nsame = 0
    for s, t in groups(w, 1e-6 * tn):
        if t - s == 1:
            a = np.sort(np.abs(Zo[:, s]))
            if a[-2] < a[-1] * (1 - 1e-8):
                assert np.abs(Zg[:, s] - Zo[:, s]).max() <= TOL_VEC
                nsame += 1
    # (every Laplacian vector has mirror-image maxima |v_i| = |v_{n+1-i}|, so nsame is 0 here;
    # the sign rule itself is checked on cfg2 below, where the maxima are unique)
    assert nsame == 0
    big = np.abs(Zg).max(axis=0)
    assert (Zg.max(axis=0) >= big * (1 - 1e-12)).all()       # a largest-|entry| is positive


def test_sign_rule_identity_cfg2(handle, torch):
    """Reading 15: with a unique largest |entry| the canonical sign makes determined vectors
    identical (no sign freedom): every P3-isolated vector of cfg2 (n = 2000) whose top two
    |entries| differ by more than 1e-8 relative matches the oracle without a sign flip."""
    d, e, w = W.problem("cfg2")
    Zg, Zo, rep = full_parity(handle, torch, d, e, w)
    tn = O.tnorm(d, e)
    nsame = niso = 0
    for s, t in groups(w, 1e-6 * tn):
        if t - s == 1:
            niso += 1
            a = np.sort(np.abs(Zo[:, s]))
            if a[-2] < a[-1] * (1 - 1e-8):
                assert np.abs(Zg[:, s] - Zo[:, s]).max() <= TOL_VEC
                nsame += 1
    assert niso >= 1900 and nsame >= 0.95 * niso, (niso, nsame)


def test_cfg2_random_full(handle, torch):
    d, e, w = W.problem("cfg2")
    full_parity(handle, torch, d, e, w)


def test_cfg3_glued_wilkinson_full(handle, torch):
    d, e, w = W.problem("cfg3")
    full_parity(handle, torch, d, e, w)


@pytest.mark.parametrize("cfg,n", [("cfg3", 1050), ("cfg4", 600), ("cfg5", 1500), ("type1", 2100),
                                   ("type2", 700), ("type3", 1050)])
def test_scaled_configs_full(handle, torch, cfg, n):
    d, e, w = W.problem(cfg, n)
    full_parity(handle, torch, d, e, w)


def test_cfg4_giant_cluster_full_size(handle, torch):
    d, e, w = W.problem("cfg4")
    Zg, rc = run_gpu(handle, torch, d, e, w)
    assert rc == 0
    res, orth = invariants_gpu(torch, d, e, w, Zg)
    assert res <= 10.0 and orth <= 10.0
    # sampled columns: the oracle's first K vectors of the (single) cluster; individual
    # vectors of cfg4 are ill-determined (gaps < 1e-8 ||T||), so report, do not gate
    K = 48
    Zo, info = O.eigvecs(d, e, w, seed=1, j_lo=0, j_hi=K)
    diff = max(vec_diff_upto_sign(Zg[:, k].cpu().numpy(), Zo[:, k]) for k in range(K))
    print(f"cfg4 sampled per-vector diff (reported) {diff:.3e}")


GOLDEN_CFG5 = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cfg5_oracle_cols.npz")


def test_cfg5_perturbed_laplacian_full_size(handle, torch):
    d, e, w = W.problem("cfg5")
    g = np.load(GOLDEN_CFG5) if os.path.exists(GOLDEN_CFG5) else None
    if g is not None:
        # the golden columns were computed from this exact w (LAPACK builds may differ in ulps)
        assert np.abs(g["w"] - w).max() <= 1e3 * EPS * O.tnorm(d, e)
        w = np.ascontiguousarray(g["w"])
        assert g["w_sha"].item().decode() == hashlib.sha256(w.tobytes()).hexdigest()
    Zg, rc = run_gpu(handle, torch, d, e, w)
    assert rc == 0
    res, orth = invariants_gpu(torch, d, e, w, Zg)
    assert res <= 10.0 and orth <= 10.0
    K = 96
    Zo, info = O.eigvecs(d, e, w, seed=1, j_lo=0, j_hi=K)
    Zs = Zg[:, :K].cpu().numpy()
    tn = O.tnorm(d, e)
    for s, t in groups(w[:K], 1e-6 * tn):
        if t == K:       # a run that may continue past the sample is not complete
            continue
        if t - s == 1:
            assert vec_diff_upto_sign(Zs[:, s], Zo[:, s]) <= TOL_VEC
        else:
            assert sigma_min(Zs[:, s:t], Zo[:, s:t]) >= 1 - TOL_SUB
    # columns across the whole chain from the full oracle run (tests/golden/make_cfg5_golden.py,
    # written by the oracle alone): P1/P3 per vector where the tau_v groups are singletons,
    # subspaces for the runs stored whole (the top run [15948, 16000))
    if g is None:
        pytest.skip("tests/golden/cfg5_oracle_cols.npz not generated")
    assert int(g["info"]) == 0
    cols = [int(c) for c in g["cols"]]
    pos = {c: k for k, c in enumerate(cols)}
    Zc = Zg[:, torch.tensor(cols, device=Zg.device)].cpu().numpy()
    nvec = nsub = 0
    for s, t in groups(w, 1e-6 * tn):
        if not all(c in pos for c in range(s, t)):
            continue
        ks = [pos[c] for c in range(s, t)]
        if t - s == 1:
            assert vec_diff_upto_sign(Zc[:, ks[0]], g["Z"][:, ks[0]]) <= TOL_VEC, s
            nvec += 1
        else:
            assert sigma_min(Zc[:, ks], g["Z"][:, ks]) >= 1 - TOL_SUB, (s, t)
            nsub += 1
    assert nvec >= 20 and nsub >= 1, (nvec, nsub)


# ------------------------------------------------------------------ edge cases

@pytest.mark.parametrize("n", [2, 3, 5, 31, 33, 37, 129, 1001])
def test_ragged_sizes(handle, torch, n):
    d, e, w = W.problem("type1", n, seed=n)
    full_parity(handle, torch, d, e, w)


def test_n1_and_zero_matrix(handle, torch):
    Z, rc = run_gpu(handle, torch, np.array([3.0]), np.zeros(0), np.array([3.0]))
    assert rc == 0 and Z.cpu().numpy().tolist() == [[1.0]]
    Z, rc = run_gpu(handle, torch, np.zeros(5), np.zeros(4), np.zeros(5))
    assert rc == 0 and np.array_equal(Z.cpu().numpy(), np.eye(5))


def test_diagonal_and_split_matrix(handle, torch):
    d = np.array([3.0, -1.0, 2.0, 7.0, 0.5])
    w = np.sort(d)
    full_parity(handle, torch, d, np.zeros(4), w)
    # a zero off-diagonal splits T into blocks
    d, e = W.random_sym(300, 7)
    e[100] = 0.0
    e[200] = 0.0
    full_parity(handle, torch, d, e, W.eigenvalues(d, e))


def test_exact_duplicates(handle, torch):
    # two identical decoupled W21+ blocks: every eigenvalue exactly duplicated
    d, e = W.glued_wilkinson(2, 0.0)
    full_parity(handle, torch, d, e, W.eigenvalues(d, e))


def _iters_of(handle):
    return handle.stats()["iters_hist"]


def test_restart_branch(handle, torch):
    """Reading 16 on the device: T = diag(1, 2), w = [1, 1] (one cluster of 2).  The second
    vector's first iterate lies in span(z_0): the compact-WY step restarts it with the start
    vector of restart 1.  Same Z (= I up to rounding), return code and iteration counts as
    the oracle (test_oracle.py::test_restart_branch_closed_form pins the oracle)."""
    d, e, w = np.array([1.0, 2.0]), np.array([0.0]), np.array([1.0, 1.0])
    Zg, rc = run_gpu(handle, torch, d, e, w)
    Zo, info, its = O.eigvecs(d, e, w, seed=1, return_iters=True)
    assert rc == info == 0
    assert np.abs(Zg.cpu().numpy() - Zo).max() <= 1e-14
    assert np.abs(Zg.cpu().numpy() - np.eye(2)).max() <= 1e-14
    hist = _iters_of(handle)
    assert hist == list(np.bincount(its, minlength=8)[:8]), (hist, its)


def test_restart_exhausted_inside_larger_cluster(handle, torch):
    """Restarts in a wider cluster, run on the resident (narrow) kernel and on the persistent
    one: T = diag(1, 200, 300, 400, 500, 600) with three shifts on eigenvalue 1.  Vector 1's
    iterates stay in span(z_0) (the other components are damped by ~1/200 against 1/(10 eps)),
    so it restarts twice, then is kept and flagged (reading 16: rc = 1); vector 2 is accepted.
    Same Z, rc and iteration histogram as the oracle."""
    d = np.array([1.0, 200.0, 300.0, 400.0, 500.0, 600.0])
    e = np.zeros(5)
    w = np.array([1.0, 1.0, 1.0, 400.0, 500.0, 600.0])
    Zo, info, its = O.eigvecs(d, e, w, seed=1, return_iters=True)
    assert info == 1 and its[1] > 2, (info, its)          # the oracle restarts and flags
    for resident in (True, False):
        handle.set_resident(resident)
        try:
            Zg, rc = run_gpu(handle, torch, d, e, w)
            hist = _iters_of(handle)
        finally:
            handle.set_resident(True)
        assert rc == info, (resident, rc, info)
        assert np.abs(Zg.cpu().numpy() - Zo).max() <= 1e-10, resident
        assert hist == list(np.bincount(its, minlength=8)[:8]), (resident, hist, its)


def test_maxits_flag(handle, torch):
    """Readings 9/17 on the device: tiny-scale diagonal T with shifts far from every eigenvalue
    (the oracle pin test_maxits_flag_closed_form proves no iterate can pass the growth test):
    every vector runs MAXITS = 5 iterations and is counted in the return code; the kept
    iterates equal the oracle's."""
    s = 1e-20
    d = s * np.array([1.0, 3.0, 5.0, 5.002, 5.004])
    e = np.zeros(4)
    w = s * np.array([2.0, 3.6, 6.0, 6.0 + 1e-6, 6.0 + 2e-6])
    Zo, info, its = O.eigvecs(d, e, w, seed=1, return_iters=True)
    Zg, rc = run_gpu(handle, torch, d, e, w)
    assert info == 5 and rc == 5, (rc, info)
    assert _iters_of(handle)[5] == 5
    assert np.abs(Zg.cpu().numpy() - Zo).max() <= 1e-10


@pytest.mark.parametrize("k", [-1000, -500, -150, 150, 300])
@pytest.mark.parametrize("cfg,n", [("cfg2", 300), ("cfg3", 210), ("cfg4", 200)])
def test_scaled_matrices(handle, torch, cfg, n, k):
    """T, w scaled by 2^k (exact): the eigenvectors of 2^k T are those of T.  Outside
    [2^-200, 2^200] both sides first rescale to ||T||_1 in [1, 2) (reading 21; at 2^-1000 the
    pivot floor eps ||T||_1 would be subnormal and sigma would lose its precision); +-150 run
    unscaled.  Gates: the GPU returns the oracle's code, the vectors satisfy the P0 invariants
    of the UNSCALED problem, and match the oracle's run on the scaled input per vector / per
    subspace (P1-P3)."""
    d, e, w = W.problem(cfg, n)
    s = 2.0 ** k
    ds, es, ws_ = d * s, e * s, w * s
    Zg, rc = run_gpu(handle, torch, ds, es, ws_)
    Zo, info = O.eigvecs(ds, es, ws_, seed=1)
    assert rc == info == 0, (rc, info)
    res, orth = invariants_gpu(torch, d, e, w, Zg)
    assert res <= 10.0 and orth <= 10.0, (res, orth)
    wv, wsig, _, _ = parity_report(w, O.tnorm(d, e), Zg.cpu().numpy(), Zo)
    assert wv <= TOL_VEC and wsig >= 1 - TOL_SUB, (wv, wsig)


def test_invalid_arguments(handle, torch):
    import ctypes as C

    L = handle._L
    dev = torch.device("cuda:0")
    d = torch.ones(4, dtype=torch.float64, device=dev)
    e = torch.ones(3, dtype=torch.float64, device=dev)
    w = torch.arange(4, dtype=torch.float64, device=dev)
    Z = torch.empty(16, dtype=torch.float64, device=dev)
    P = lambda t: C.c_void_p(t.data_ptr())
    assert L.tinv_eigvecs(handle._h, 0, P(d), P(e), P(w), P(Z), 4, 1) == -2
    assert L.tinv_eigvecs(handle._h, 4, None, P(e), P(w), P(Z), 4, 1) == -3
    assert L.tinv_eigvecs(handle._h, 4, P(d), None, P(w), P(Z), 4, 1) == -4
    assert L.tinv_eigvecs(handle._h, 4, P(d), P(e), P(w), P(Z), 3, 1) == -7
    bad = d.clone()
    bad[2] = float("nan")
    assert L.tinv_eigvecs(handle._h, 4, P(bad), P(e), P(w), P(Z), 4, 1) == -3
    wdesc = torch.tensor([3.0, 2.0, 1.0, 0.0], dtype=torch.float64, device=dev)
    assert L.tinv_eigvecs(handle._h, 4, P(d), P(e), P(wdesc), P(Z), 4, 1) == -5
    assert L.tinv_eigvecs(None, 4, P(d), P(e), P(w), P(Z), 4, 1) == -103


def test_ldz_larger_than_n(handle, torch):
    import ctypes as C

    d, e, w = W.problem("cfg2", 300)
    n, ldz = 300, 317
    dev = torch.device("cuda:0")
    dt, et, wt = (torch.tensor(a, dtype=torch.float64, device=dev) for a in (d, e, w))  # kept alive
    Zbuf = torch.full((n, ldz), 7.0, dtype=torch.float64, device=dev)
    rc = handle._L.tinv_eigvecs(handle._h, n, C.c_void_p(dt.data_ptr()), C.c_void_p(et.data_ptr()),
                                C.c_void_p(wt.data_ptr()), C.c_void_p(Zbuf.data_ptr()), ldz, 1)
    torch.cuda.synchronize()
    assert rc == 0
    Zb = Zbuf.cpu().numpy()
    assert (Zb[:, n:] == 7.0).all()              # padding rows untouched
    Zg, _ = run_gpu(handle, torch, d, e, w)
    assert np.array_equal(Zb[:, :n].T, Zg.cpu().numpy())


# ------------------------------------------------------------------ determinism / paths

def test_deterministic_bitwise(handle, torch):
    d, e, w = W.problem("cfg3", 840)
    Z1, _ = run_gpu(handle, torch, d, e, w)
    Z2, _ = run_gpu(handle, torch, d, e, w)
    assert torch.equal(Z1, Z2)


def test_host_path_equals_device_path(handle, torch):
    d, e, w = W.problem("cfg2", 500)
    Zd, _ = run_gpu(handle, torch, d, e, w)
    Zh, rc = handle.eigvecs_host(np.ascontiguousarray(d), np.ascontiguousarray(e), np.ascontiguousarray(w), seed=1)
    assert rc == 0
    assert np.array_equal(Zh.T, Zd.cpu().numpy())


def test_host_path_pinned_mapped_z(handle, torch):
    """Pinned (mapped) Z: the kernels write the columns straight into host memory; the result
    equals the device path bit for bit, on a resident-kernel config and a persistent one."""
    for cfg, n in (("cfg2", 800), ("cfg3", 630)):
        d, e, w = W.problem(cfg, n)
        Zd, _ = run_gpu(handle, torch, d, e, w)
        hd, he, hw = (torch.tensor(a, dtype=torch.float64).pin_memory() for a in (d, e, w))
        hZ = torch.full((n, n), float("nan"), dtype=torch.float64).pin_memory()
        Zh, rc = handle.eigvecs_host(hd, he, hw, Z=hZ, seed=1)
        assert rc == 0
        assert torch.equal(hZ, Zd.cpu().t())   # hZ row j = column j (column-major Z)


def test_stats_report_native_launches(handle, torch):
    d, e, w = W.problem("cfg2", 400)
    run_gpu(handle, torch, d, e, w)
    st = handle.stats()
    assert st["launches"] >= 3 and st["n"] == 400 and st["nclusters"] >= 1
    assert sum(st["iters_hist"]) == 400


# ------------------------------------------------------------------ eigenvalues

@pytest.mark.parametrize("cfg,n", [("cfg1", None), ("cfg2", None), ("cfg3", 1050), ("cfg4", 600), ("cfg5", 1500),
                                   ("type1", 333), ("type2", 257), ("type3", 105)])
def test_bisection_bit_exact(handle, torch, cfg, n):
    """Sturm counts are integers decided by floating point: the GPU takes every decision in
    the oracle's arithmetic (explicit round-to-nearest, no contraction), so the eigenvalues are
    identical bit for bit."""
    d, e = W.make(cfg, n)
    dev = torch.device("cuda:0")
    w = handle.eigvals(torch.tensor(d, device=dev), torch.tensor(e, device=dev)).cpu().numpy()
    wo = O.bisect(d, e)
    assert np.array_equal(w, wo), np.abs(w - wo).max()


def test_bisection_edge_cases(handle, torch):
    dev = torch.device("cuda:0")
    w = handle.eigvals(torch.tensor([3.5], dtype=torch.float64, device=dev), torch.zeros(0, dtype=torch.float64,
                                                                                         device=dev))
    assert w.cpu().numpy().tolist() == O.bisect(np.array([3.5]), np.zeros(0)).tolist()
    for d, e in ((np.zeros(7), np.zeros(6)), (np.array([1.0, 1.0, 1.0]), np.zeros(2)),
                 (np.full(40, 2.0), np.full(39, -1.0))):
        w = handle.eigvals(torch.tensor(d, device=dev), torch.tensor(e, device=dev)).cpu().numpy()
        assert np.array_equal(w, O.bisect(d, e))


def test_bisection_full_size_cfg5(handle, torch):
    d, e = W.make("cfg5")
    dev = torch.device("cuda:0")
    w = handle.eigvals(torch.tensor(d, device=dev), torch.tensor(e, device=dev)).cpu().numpy()
    assert np.all(np.diff(w) >= 0)
    # sampled indices: the oracle's Sturm count brackets each w_k within a few ulps
    tn = O.tnorm(d, e)
    for k in (0, 1, 777, 8000, 15998, 15999):
        dx = 8 * np.spacing(max(abs(w[k]), tn * 1e-300))
        assert O.sturm_count(d, e, w[k] - dx, tn) <= k < O.sturm_count(d, e, w[k] + dx, tn)


def test_eig_end_to_end(handle, torch):
    """T -> (w, Z) entirely on the device: eigenvalues by bisection then DSTEIN-cWY."""
    d, e = W.make("cfg2", 700)
    dev = torch.device("cuda:0")
    w, Z, rc = handle.eig(torch.tensor(d, device=dev), torch.tensor(e, device=dev))
    torch.cuda.synchronize()
    assert rc == 0
    wh = w.cpu().numpy()
    assert np.array_equal(wh, O.bisect(d, e))
    res, orth = invariants_gpu(torch, d, e, wh, Z)
    assert res <= 10.0 and orth <= 10.0
    Zo, info = O.eigvecs(d, e, wh, seed=1)
    wv, ws, _, _ = parity_report(wh, O.tnorm(d, e), Z.cpu().numpy(), Zo)
    assert wv <= TOL_VEC and ws >= 1 - TOL_SUB


# ------------------------------------------------------------------ multi-GPU row split

@pytest.mark.parametrize("vr", [2, 3, 4])
@pytest.mark.parametrize("cfg,n", [("cfg4", 600), ("cfg5", 1500), ("type2", 700)])
def test_row_split_virtual_ranks(handle, torch, cfg, n, vr):
    """One giant cluster split over `vr` virtual ranks (groups of one launch with their own
    workspace replicas, mirrored stores, partial sums read from the owner's replica, the
    rank-replicated barrier): the same code path as real ranks over NVLink.  Parity with the
    oracle (P0 invariants, P1/P3 per-vector and subspace agreement)."""
    d, e, w = W.problem(cfg, n)
    handle.set_virtual_ranks(vr)
    try:
        full_parity(handle, torch, d, e, w)
        st = handle.stats()
    finally:
        handle.set_virtual_ranks(1)
    cs = O.clusters(w, O.tnorm(d, e))
    big = [b - a for a, b in zip(cs[:-1], cs[1:]) if b - a > 1]
    if len(big) == 1 and big[0] > 64:
        assert st["ngroups"] == vr          # the cluster really ran row-split


def test_row_split_virtual_ranks_full_size_cfg4(handle, torch):
    d, e, w = W.problem("cfg4")
    handle.set_virtual_ranks(2)
    try:
        Zg, rc = run_gpu(handle, torch, d, e, w)
        st = handle.stats()
    finally:
        handle.set_virtual_ranks(1)
    assert rc == 0 and st["ngroups"] == 2
    res, orth = invariants_gpu(torch, d, e, w, Zg)
    assert res <= 10.0 and orth <= 10.0


# ------------------------------------------------------------------ resident (DSMEM) compact-WY path

def _clustered(n, sizes, seed=3):
    """Tridiagonal with planted Peters-Wilkinson clusters of the given sizes; the remaining
    vectors form clusters of 3 or 6 (with n > 1000 every spectrum has clusters under the
    1e-3 ||T||_1 rule).  Groups sit 1 apart, their members within 1e-7; e is tiny."""
    rng = np.random.default_rng(seed)
    groups = list(sizes)
    rest = n - sum(sizes)
    f = 3 if n <= 2500 else 6   # fewer than ~900 groups keep them 1e-3 ||T||_1 apart
    groups += [f] * (rest // f) + ([rest % f] if rest % f else [])
    rng.shuffle(groups)
    d = np.concatenate([g + 1e-7 * rng.uniform(-1, 1, m) for g, m in enumerate(groups)])
    e = 1e-9 * rng.uniform(-1, 1, n - 1)
    return d, e, W.eigenvalues(d, e)


@pytest.mark.parametrize("n,sizes", [(2000, [60, 33, 17, 9, 2]), (1999, [64, 5, 3]), (1501, [40, 12, 7]),
                                     (4096, [48, 24, 2])])
def test_resident_cluster_sizes(handle, torch, n, sizes):
    """Clusters needing 1, 2, 4 and 8 CTAs of a thread-block cluster (m up to 64), odd n."""
    d, e, w = _clustered(n, sizes)
    cs = O.clusters(w, O.tnorm(d, e))
    assert max(np.diff(cs)) == max(sizes)
    Zg, Zo, rep = full_parity(handle, torch, d, e, w)
    assert handle.stats()["resident_groups"] >= 1


def test_resident_equals_streaming_path(handle, torch):
    """The resident kernel and the streaming persistent kernel compute the same vectors (up to
    rounding) on the many-small-clusters workload."""
    d, e, w = W.problem("cfg2", 1200)
    dev = torch.device("cuda:0")
    Zr, rc = run_gpu(handle, torch, d, e, w)
    assert handle.stats()["resident_groups"] >= 1
    handle.set_resident(False)
    try:
        Zs, rc2 = run_gpu(handle, torch, d, e, w)
        assert handle.stats()["resident_groups"] == 0
    finally:
        handle.set_resident(True)
    assert rc == 0 and rc2 == 0
    wv, ws, _, _ = parity_report(w, O.tnorm(d, e), Zr.cpu().numpy(), Zs.cpu().numpy())
    assert wv <= TOL_VEC and ws >= 1 - TOL_SUB


def test_resident_deterministic(handle, torch):
    d, e, w = W.problem("cfg2")
    Z1, _ = run_gpu(handle, torch, d, e, w)
    Z2, _ = run_gpu(handle, torch, d, e, w)
    assert torch.equal(Z1, Z2)


# ------------------------------------------------------------------ Alg. 1 (classical MGS)
# tinv_set_reorth(h, 1) -- modified Gram-Schmidt against the cluster's
# accepted vectors in the resident kernel, compared with the MGS oracle.

def _mgs_parity(handle, torch, d, e, w):
    handle.set_reorth("mgs")
    try:
        Zg, rc = run_gpu(handle, torch, d, e, w)
    finally:
        handle.set_reorth("cwy")
    assert rc == 0, f"tinv_eigvecs (MGS) returned {rc}"
    res, orth = invariants_gpu(torch, d, e, w, Zg)
    assert res <= 10.0 and orth <= 10.0
    Zo, info = O.eigvecs(d, e, w, seed=1, mgs=True)
    assert info == 0
    Zg_h = Zg.cpu().numpy()
    wv, ws, nv, ng = parity_report(w, O.tnorm(d, e), Zg_h, Zo)
    assert wv <= TOL_VEC and ws >= 1 - TOL_SUB
    return Zg_h


@pytest.mark.parametrize("cfg,n", [("cfg2", 1200), ("cfg1", None), ("type3", 420)])
def test_mgs_path_parity(handle, torch, cfg, n):
    d, e, w = W.problem(cfg, n)
    _mgs_parity(handle, torch, d, e, w)


@pytest.mark.parametrize("n,sizes", [(2000, [60, 33, 17, 9, 2]), (1501, [40, 12, 7])])
def test_mgs_cluster_sizes(handle, torch, n, sizes):
    """1- to 8-CTA thread-block clusters, m up to 60: MGS vs its oracle, and vs the cWY path."""
    d, e, w = _clustered(n, sizes)
    Zm = _mgs_parity(handle, torch, d, e, w)
    Zc, rc = run_gpu(handle, torch, d, e, w)
    assert rc == 0
    wv, ws, _, _ = parity_report(w, O.tnorm(d, e), Zm, Zc.cpu().numpy())
    assert wv <= TOL_VEC and ws >= 1 - TOL_SUB


@pytest.mark.parametrize("cfg,n", [("cfg4", 600), ("type2", 700), ("cfg3", 1050), ("type1", 2100)])
def test_mgs_wide_clusters(handle, torch, cfg, n):
    """Clusters too wide for the resident kernel run MGS in the persistent kernel (one group
    barrier per accepted vector, small CTA groups): parity with the MGS oracle (Alg. 1) and,
    where the vectors are determined, with the compact-WY path."""
    d, e, w = W.problem(cfg, n)
    Zm = _mgs_parity(handle, torch, d, e, w)
    Zc, rc = run_gpu(handle, torch, d, e, w)
    assert rc == 0
    wv, ws, _, _ = parity_report(w, O.tnorm(d, e), Zm, Zc.cpu().numpy())
    assert wv <= TOL_VEC and ws >= 1 - TOL_SUB


@pytest.mark.parametrize("mode", ["mgs", "ordinary"])
def test_reorth_modes_restart_persistent(handle, torch, mode):
    """Reading 16 in the persistent kernel's comparison modes (set_resident(False) puts the
    narrow cluster there): T = diag(1, 200, .., 600) with three shifts on eigenvalue 1 --
    vector 1 restarts twice and is flagged on both sides (rc = 1), the same Z and iteration
    histogram as the oracle of that mode (MGS: Alg. 1; ordinary: the compact-WY oracle)."""
    d = np.array([1.0, 200.0, 300.0, 400.0, 500.0, 600.0])
    e = np.zeros(5)
    w = np.array([1.0, 1.0, 1.0, 400.0, 500.0, 600.0])
    Zo, info, its = O.eigvecs(d, e, w, seed=1, return_iters=True, mgs=(mode == "mgs"))
    assert info == 1 and its[1] > 2, (info, its)
    handle.set_resident(False)
    handle.set_reorth(mode)
    try:
        Zg, rc = run_gpu(handle, torch, d, e, w)
        hist = _iters_of(handle)
    finally:
        handle.set_reorth("cwy")
        handle.set_resident(True)
    assert rc == info, (rc, info)
    assert hist == list(np.bincount(its, minlength=8)[:8]), (hist, its)
    Zh = Zg.cpu().numpy()
    # MGS: the kept iterate of the flagged vector 1 is x - <x, z_0> z_0 with x ~ 1e15 e_0, i.e.
    # rounding noise in the e_0 direction (one Gram-Schmidt projection of a vector inside the
    # span); it and vector 2 (projected against it) are not determined -- only unit norm.
    # The compact-WY step forms q = Y x' - e_p instead and agrees to 1e-10 everywhere.
    cols = [0, 3, 4, 5] if mode == "mgs" else range(6)
    for k in cols:
        assert np.abs(Zh[:, k] - Zo[:, k]).max() <= 1e-10, k
    assert np.abs(np.linalg.norm(Zh, axis=0) - 1).max() <= 1e-14


@pytest.mark.parametrize("mode", ["mgs", "ordinary"])
@pytest.mark.parametrize("cfg,n", [("cfg2", 1200), ("cfg1", None)])
def test_reorth_modes_persistent_narrow(handle, torch, mode, cfg, n):
    """The comparison modes' persistent-kernel code for narrow clusters (m <= 64, forced off
    the resident kernel) against the oracle of the mode."""
    d, e, w = W.problem(cfg, n)
    handle.set_resident(False)
    handle.set_reorth(mode)
    try:
        Zg, rc = run_gpu(handle, torch, d, e, w)
    finally:
        handle.set_reorth("cwy")
        handle.set_resident(True)
    assert rc == 0
    res, orth = invariants_gpu(torch, d, e, w, Zg)
    assert res <= 10.0 and orth <= 10.0
    Zo, info = O.eigvecs(d, e, w, seed=1, mgs=(mode == "mgs"))
    wv, ws, _, _ = parity_report(w, O.tnorm(d, e), Zg.cpu().numpy(), Zo)
    assert wv <= TOL_VEC and ws >= 1 - TOL_SUB


def test_reorth_modes_unsupported_for_row_split(handle, torch):
    from paper_1209_1910_b200.tinv import TinvError

    d, e, w = W.problem("cfg4", 600)      # one wide cluster, split over 2 virtual ranks
    handle.set_virtual_ranks(2)
    try:
        for mode in ("mgs", "ordinary"):
            handle.set_reorth(mode)
            try:
                with pytest.raises(TinvError, match="-105"):
                    run_gpu(handle, torch, d, e, w)
            finally:
                handle.set_reorth("cwy")
    finally:
        handle.set_virtual_ranks(1)
    Z, rc = run_gpu(handle, torch, d, e, w)   # the handle still works in cWY mode
    assert rc == 0


# ------------------------------------------------------------------ §3.3.1 ordinary sequence
# tinv_set_reorth(h, 2) -- the same compact-WY step in the ordinary BLAS
# sequence (Y^T y by its own pass); equals the compact-WY oracle within tolerance.

@pytest.mark.parametrize("cfg,n,sizes", [("cfg2", 1200, None), ("clustered", 2000, [60, 33, 17, 9, 2]),
                                         ("type3", 420, None), ("cfg4", 600, None), ("type2", 700, None),
                                         ("cfg3", 1050, None), ("clustered", 5000, [300, 40, 9])])
def test_ordinary_cwy_path_parity(handle, torch, cfg, n, sizes):
    d, e, w = _clustered(n, sizes) if sizes else W.problem(cfg, n)
    handle.set_reorth("ordinary")
    try:
        Zg, rc = run_gpu(handle, torch, d, e, w)
    finally:
        handle.set_reorth("cwy")
    assert rc == 0
    res, orth = invariants_gpu(torch, d, e, w, Zg)
    assert res <= 10.0 and orth <= 10.0
    Zo, info = O.eigvecs(d, e, w, seed=1)
    wv, ws, _, _ = parity_report(w, O.tnorm(d, e), Zg.cpu().numpy(), Zo)
    assert wv <= TOL_VEC and ws >= 1 - TOL_SUB


@pytest.mark.parametrize("mode", ["mgs", "ordinary"])
def test_reorth_modes_without_handover(handle, torch, mode):
    """n > 2048: the batched LU iterates every leader (no handover); the resident kernel reads
    them from Z.  Both comparison modes against their oracle."""
    d, e, w = _clustered(3000, [20, 12, 7])   # clusters that fit the resident kernel at n = 3000
    handle.set_reorth(mode)
    try:
        Zg, rc = run_gpu(handle, torch, d, e, w)
        assert handle.stats()["resident_groups"] >= 1
    finally:
        handle.set_reorth("cwy")
    assert rc == 0
    res, orth = invariants_gpu(torch, d, e, w, Zg)
    assert res <= 10.0 and orth <= 10.0
    Zo, info = O.eigvecs(d, e, w, seed=1, mgs=(mode == "mgs"))
    wv, ws, _, _ = parity_report(w, O.tnorm(d, e), Zg.cpu().numpy(), Zo)
    assert wv <= TOL_VEC and ws >= 1 - TOL_SUB


# ------------------------------------------------------------------ blocked look-ahead
# tinv_set_lookahead(h, b) -- the first iterates of each block of b vectors
# get the accepted reflectors applied at once (two skinny GEMMs + a TRMM); same results as the
# per-vector step up to rounding: parity with the compact-WY oracle.

@pytest.mark.parametrize("b", [2, 5, 8])
@pytest.mark.parametrize("cfg,n", [("cfg4", 600), ("type2", 700), ("cfg3", 1050), ("cfg5", 1500)])
def test_blocked_lookahead_parity(handle, torch, cfg, n, b):
    d, e, w = W.problem(cfg, n)
    handle.set_lookahead(b)
    try:
        Zg, rc = run_gpu(handle, torch, d, e, w)
    finally:
        handle.set_lookahead(0)
    assert rc == 0
    res, orth = invariants_gpu(torch, d, e, w, Zg)
    assert res <= 10.0 and orth <= 10.0
    Zo, info = O.eigvecs(d, e, w, seed=1)
    wv, ws, _, _ = parity_report(w, O.tnorm(d, e), Zg.cpu().numpy(), Zo)
    assert wv <= TOL_VEC and ws >= 1 - TOL_SUB


def test_blocked_lookahead_restarts(handle, torch):
    """Block vectors that restart (reading 16), in the reduced and the ordinary sequence:
    T = diag(1, 200, 201, ..) (n = 80) with 70 shifts on eigenvalue 1 -- one cluster of 70, so
    vectors 65..69 take the block path; their iterates stay in span(z_0) and restart (the
    oracle flags 54 vectors).  Same return code and iteration histogram as the oracle."""
    d = np.concatenate([[1.0], 200.0 + np.arange(79.0)])
    e = np.zeros(79)
    w = np.concatenate([[1.0] * 70, d[70:]])
    Zo, info, its = O.eigvecs(d, e, w, seed=1, return_iters=True)
    assert info > 0 and (its[65:70] > 2).all(), (info, its[60:75])
    for md in ("cwy", "ordinary"):
        handle.set_lookahead(4)
        handle.set_reorth(md)
        try:
            Zg, rc = run_gpu(handle, torch, d, e, w)
            hist = _iters_of(handle)
        finally:
            handle.set_reorth("cwy")
            handle.set_lookahead(0)
        assert rc == info, (md, rc, info)
        assert hist == list(np.bincount(its, minlength=8)[:8]), (md, hist, its)
        assert np.abs(np.linalg.norm(Zg.cpu().numpy(), axis=0) - 1).max() <= 1e-14


def test_blocked_lookahead_full_size_cfg4(handle, torch):
    d, e, w = W.problem("cfg4")
    handle.set_lookahead(8)
    try:
        Zg, rc = run_gpu(handle, torch, d, e, w)
    finally:
        handle.set_lookahead(0)
    assert rc == 0
    res, orth = invariants_gpu(torch, d, e, w, Zg)
    assert res <= 10.0 and orth <= 10.0


@pytest.mark.parametrize("vr", [2, 3])
def test_row_split_virtual_ranks_mixed(handle, torch, vr):
    """A dominant wide cluster (700 of 3000 vectors) plus a wide one of 100 and many small ones: the big cluster is
    row-split over `vr` virtual ranks while the others run as ordinary groups (and narrow ones
    in the resident kernel) in the same launch -- SURVEY §8(e) regime 2 next to regime 1.
    Parity with the oracle."""
    d, e, w = _clustered(3000, [700, 100, 9])
    handle.set_virtual_ranks(vr)
    try:
        full_parity(handle, torch, d, e, w)
        st = handle.stats()
    finally:
        handle.set_virtual_ranks(1)
    assert st["ngroups"] >= vr + 1, st["ngroups"]     # vr split groups + the other clusters' groups


# ------------------------------------------------------------------ deferred final pass D
# the last iteration's pass D (q = Y_{p+1} x' - e_p) of a wide
# cluster's vector is formed after the cWY kernel by one GEMM (dz.cu) from the parked x'; Y and
# T are bitwise those of the per-vector path, so only the parked columns' summation order
# differs.  A failed deferred stopping test re-runs the call without deferral.

def _run_dz(handle, torch, d, e, w, dz, env=None):
    handle.set_deferred(dz)
    old = os.environ.get("TINV_DZ")
    if env is not None:
        os.environ["TINV_DZ"] = env
    try:
        Z, rc = run_gpu(handle, torch, d, e, w)
        st = handle.stats()
    finally:
        handle.set_deferred(True)
        if env is not None:
            if old is None:
                del os.environ["TINV_DZ"]
            else:
                os.environ["TINV_DZ"] = old
    return Z, rc, st


@pytest.mark.parametrize("b", [0, 8])
@pytest.mark.parametrize("cfg,n", [("cfg4", 600), ("cfg3", 1050), ("cfg5", 1500), ("type2", 700), ("cfg4", 1999)])
def test_deferred_pass_d_parity(handle, torch, cfg, n, b):
    d, e, w = W.problem(cfg, n)
    handle.set_lookahead(b)
    try:
        Zd, rc, st = _run_dz(handle, torch, d, e, w, True)
        Zn, rc2, st2 = _run_dz(handle, torch, d, e, w, False)
    finally:
        handle.set_lookahead(0)
    assert rc == 0 and rc2 == 0
    assert st["dz_parked"] > 0 and st["dz_redo"] == 0, st
    assert st2["dz_parked"] == 0
    assert st["iters_hist"] == st2["iters_hist"]
    Zd_h, Zn_h = Zd.cpu().numpy(), Zn.cpu().numpy()
    diff = np.minimum(np.abs(Zd_h - Zn_h).max(axis=0), np.abs(Zd_h + Zn_h).max(axis=0)).max()
    assert diff <= 1e-12, diff
    res, orth = invariants_gpu(torch, d, e, w, Zd)
    assert res <= 10.0 and orth <= 10.0
    Zo, info = O.eigvecs(d, e, w, seed=1)
    wv, ws, _, _ = parity_report(w, O.tnorm(d, e), Zd_h, Zo)
    assert wv <= TOL_VEC and ws >= 1 - TOL_SUB


def test_deferred_pass_d_forced_rerun(handle, torch):
    """TINV_DZ=2 treats every parked vector as failed: the call re-runs without deferral and
    returns exactly the per-vector path's Z."""
    d, e, w = W.problem("cfg4", 800)
    handle.set_lookahead(8)
    try:
        Zf, rc, st = _run_dz(handle, torch, d, e, w, True, env="2")
        Zn, rc2, _ = _run_dz(handle, torch, d, e, w, False)
    finally:
        handle.set_lookahead(0)
    assert rc == 0 and rc2 == 0
    assert st["dz_redo"] == -1 and st["dz_parked"] == 0, st
    assert torch.equal(Zf, Zn)


def test_deferred_pass_d_restarts_and_flags(handle, torch):
    """The restart / MAXITS fixture of test_blocked_lookahead_restarts with the deferral on:
    same return code and iteration histogram as the oracle, whether or not a deferred test
    failed (then the call re-ran without deferral)."""
    d = np.concatenate([[1.0], 200.0 + np.arange(79.0)])
    e = np.zeros(79)
    w = np.concatenate([[1.0] * 70, d[70:]])
    Zo, info, its = O.eigvecs(d, e, w, seed=1, return_iters=True)
    for b in (0, 4):
        handle.set_lookahead(b)
        try:
            Zg, rc, st = _run_dz(handle, torch, d, e, w, True)
            hist = _iters_of(handle)
        finally:
            handle.set_lookahead(0)
        assert rc == info, (b, rc, info, st["dz_redo"])
        assert hist == list(np.bincount(its, minlength=8)[:8]), (b, hist)
        assert np.abs(np.linalg.norm(Zg.cpu().numpy(), axis=0) - 1).max() <= 1e-14


def test_deferred_pass_d_full_size_cfg4(handle, torch):
    d, e, w = W.problem("cfg4")
    handle.set_lookahead(8)
    try:
        Zg, rc, st = _run_dz(handle, torch, d, e, w, True)
    finally:
        handle.set_lookahead(0)
    assert rc == 0 and st["dz_parked"] > 7000 and st["dz_redo"] == 0, st
    res, orth = invariants_gpu(torch, d, e, w, Zg)
    assert res <= 10.0 and orth <= 10.0


@pytest.mark.parametrize("cfg,n", [("cfg4", 900), ("cfg5", 1500), ("type1", 1050)])
def test_pass_d_cta0_share(handle, torch, cfg, n):
    """TINV_CTA0 (per-mille cut of CTA 0's share of pass D's rows, default 120) only moves whole
    rows of the row-dot pass D -- and with them the CTA pieces of the partitioned forward sweep --
    between CTAs: same iteration counts, Z equal to rounding, invariants and oracle parity at
    every setting."""
    d, e, w = W.problem(cfg, n)
    dd, de, dw = (torch.tensor(x, dtype=torch.float64, device="cuda:0") for x in (d, e, w))
    old = os.environ.get("TINV_CTA0")
    out = {}
    try:
        for v in ("0", "120", "600"):
            os.environ["TINV_CTA0"] = v
            Z, rc = handle.eigvecs(dd, de, dw, seed=1)
            out[v] = (Z.clone(), rc, handle.stats()["iters_hist"])
    finally:
        if old is None:
            del os.environ["TINV_CTA0"]
        else:
            os.environ["TINV_CTA0"] = old
    Zo, info = O.eigvecs(d, e, w, seed=1)
    for v, (Z, rc, hist) in out.items():
        assert rc == 0 and hist == out["0"][2], (v, rc, hist)
        res, orth = invariants_gpu(torch, d, e, w, Z)
        assert res <= 10.0 and orth <= 10.0, (v, res, orth)
        wv, ws, _, _ = parity_report(w, O.tnorm(d, e), Z.cpu().numpy(), Zo)
        assert wv <= TOL_VEC and ws >= 1 - TOL_SUB, (v, wv, ws)
