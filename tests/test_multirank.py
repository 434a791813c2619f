"""Multi-rank (N > 1) host logic on CPU, world_size 2 over torch.distributed `gloo`.

tinv_eigvecs with nranks > 1 shards the Peters-Wilkinson clusters (they are
independent: PAPER.md:168-171) over the ranks in the contiguous column ranges returned by the
library's own partitioner (tinv_partition, host-only), computes each rank's columns, and
broadcasts each rank's column block so every rank ends with the complete Z.  These tests run
that orchestration with two gloo processes: the partition comes from libtinv, the per-rank
column compute is the CPU oracle standing in for the GPU kernels (no device here), and the
exchange is the same per-rank block broadcast.  They check that the partition covers every
column exactly once without cutting a cluster, that it balances the reorthogonalisation
cost, and that the assembled Z equals a single-process run bit for bit (each eigenvector
depends only on its own cluster, so sharding must not change any column).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_1209_1910_b200 import tinv
from paper_1209_1910_b200 import workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(cfg, n):
    if cfg == "mixed":   # one dominant wide cluster (row split) plus small ones (sharded)
        rng = np.random.default_rng(5)
        groups = [120] + [3] * ((n - 120) // 3)
        rng.shuffle(groups)
        d = np.concatenate([g + 1e-7 * rng.uniform(-1, 1, k) for g, k in enumerate(groups)])
        e = 1e-9 * rng.uniform(-1, 1, len(d) - 1)
        return d, e, W.eigenvalues(d, e)
    return W.problem(cfg, n)


def _worker(rank, world, port, cfg, n, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        d, e, w = _problem(cfg, n)
        n = len(d)
        cs = O.clusters(w, O.tnorm(d, e))
        ranges, split = tinv.plan(cs, world)
        lo, hi = ranges[rank]
        # this rank's columns (stand-in for the GPU compute of its clusters); the row-split
        # cluster is computed by all ranks together (on the GPU: its rows split over them)
        Zloc = np.zeros((n, n))
        own = [(lo, hi)]
        if split >= 0:
            a, b = int(cs[split]), int(cs[split + 1])
            own = [(lo, min(hi, a)), (max(lo, b), hi)] if lo <= a < hi else own
            Zs, info = O.eigvecs(d, e, w, seed=1, j_lo=a, j_hi=b)
            assert info == 0
            Zloc[:, a:b] = Zs[:, a:b] if Zs.shape[1] == n else Zs
        for a, b in own:
            if b > a:
                Zr, info = O.eigvecs(d, e, w, seed=1, j_lo=a, j_hi=b)
                assert info == 0
                Zloc[:, a:b] = Zr[:, a:b] if Zr.shape[1] == n else Zr
        # exchange: every rank broadcasts its block (what the library does with NCCL), the
        # split cluster's columns excepted (complete everywhere)
        Z = torch.tensor(Zloc)
        for r, (a, b) in enumerate(ranges):
            blocks = [(a, b)]
            if split >= 0 and a <= int(cs[split]) < b:
                blocks = [(a, int(cs[split])), (int(cs[split + 1]), b)]
            for x, y in blocks:
                blk = Z[:, x:y].contiguous()
                dist.broadcast(blk, src=r)
                Z[:, x:y] = blk
        np.save(os.path.join(out_dir, f"Z{rank}.npy"), Z.numpy())
        np.save(os.path.join(out_dir, f"ranges{rank}.npy"), np.array(ranges))
        np.save(os.path.join(out_dir, f"split{rank}.npy"), np.array([split]))
    finally:
        dist.destroy_process_group()


def _run(tmp_path, cfg, n, world=2):
    port = _free_port()
    mp.spawn(_worker, args=(world, port, cfg, n, str(tmp_path)), nprocs=world, join=True)
    Zs = [np.load(tmp_path / f"Z{r}.npy") for r in range(world)]
    rs = [np.load(tmp_path / f"ranges{r}.npy") for r in range(world)]
    sp = [int(np.load(tmp_path / f"split{r}.npy")[0]) for r in range(world)]
    assert len(set(sp)) == 1                          # every rank derived the same row split
    return Zs, rs


@pytest.mark.parametrize("cfg,n", [("cfg2", 400), ("cfg3", 630), ("cfg1", 200), ("mixed", 600)])
def test_sharded_assembly_equals_single_process(tmp_path, cfg, n):
    Zs, rs = _run(tmp_path, cfg, n)
    d, e, w = _problem(cfg, n)
    Zref, info = O.eigvecs(d, e, w, seed=1)
    assert info == 0
    for r in range(len(Zs)):
        assert np.array_equal(rs[r], rs[0])          # every rank derived the same partition
        assert np.array_equal(Zs[r], Zref)            # complete Z on every rank, bit for bit


def test_partition_covers_columns_and_respects_clusters():
    d, e, w = W.problem("cfg3", 1050)
    cs = O.clusters(w, O.tnorm(d, e))
    starts = set(int(c) for c in cs)
    for nr in (1, 2, 3, 4, 8, 16):
        ranges = tinv.partition(cs, nr)
        assert len(ranges) == nr
        assert ranges[0][0] == 0 and ranges[-1][1] == len(d)
        for (a, b), (c, _) in zip(ranges[:-1], ranges[1:]):
            assert b == c                              # contiguous, disjoint, complete
        for a, b in ranges:
            assert a <= b and a in starts and b in starts   # never cuts a cluster


def test_partition_balances_reorth_cost():
    # 16 equal clusters of 10 over 4 ranks: exactly 4 clusters each
    n = 160
    cs = np.arange(0, n + 1, 10)
    ranges = tinv.partition(cs, 4)
    assert ranges == [(0, 40), (40, 80), (80, 120), (120, 160)]
    # one giant cluster cannot be split by columns: it lands on one rank -- and is row-split
    ranges = tinv.partition(np.array([0, 100]), 3)
    assert sorted(b - a for a, b in ranges) == [0, 0, 100]
    assert tinv.plan(np.array([0, 100]), 3)[1] == 0
    assert tinv.plan(np.array([0, 100]), 1)[1] == -1          # one rank: nothing to split
    assert tinv.plan(np.array([0, 60]), 2)[1] == -1           # narrow (m <= 64): never split


def test_plan_row_split_rule():
    """the costliest cluster is row-split when it is wide and worth >= 1/N of all
    the m^2 n work; the other clusters are balanced over the ranks without it."""
    # clusters 300, 100, 100, 100 (n = 600): 300^2 = 9e4 of 1.2e5 total
    cs = np.array([0, 300, 400, 500, 600])
    for nr in (2, 4, 8):
        ranges, split = tinv.plan(cs, nr)
        assert split == 0
        owned = [c for c in range(1, 4) if any(a <= cs[c] < b for a, b in ranges)]
        assert owned == [1, 2, 3]
    # four equal clusters: none is worth more than its share at N = 2 ... but is at N = 8
    cs = np.array([0, 100, 200, 300, 400])
    assert tinv.plan(cs, 2)[1] == -1
    assert tinv.plan(cs, 8)[1] == 0
    # with the split cluster excluded, the remaining three balance one per rank on 3 ranks
    ranges, split = tinv.plan(np.array([0, 300, 400, 500, 600]), 3)
    assert split == 0
    sizes = sorted(b - a for a, b in ranges)
    assert sizes[-1] <= 400                                # the big one does not weigh down a rank


def test_partition_rejects_invalid_tables():
    with pytest.raises(tinv.TinvError):
        tinv.partition(np.array([0, 5, 5, 10]), 2)       # empty cluster
    with pytest.raises(tinv.TinvError):
        tinv.partition(np.array([1, 10]), 2)             # does not start at 0
    with pytest.raises(tinv.TinvError):
        tinv.partition(np.array([0, 10]), 0)             # no ranks
