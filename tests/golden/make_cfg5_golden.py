"""Writes tests/golden/cfg5_oracle_cols.npz: selected eigenvector columns of the FULL
cfg5 problem (BASELINE.json configs[4]: n = 16000 perturbed 1D Laplacian, seed 0; start
vectors seed 1) computed by the CPU oracle (oracle/, Alg. 4 DSTEIN-cWY).

Calls only oracle/ (the method) and paper_1209_1910_b200.workloads (seeded inputs, no method
arithmetic).  cfg5 is one cluster of 16000 vectors: column j depends on every accepted
column before it, so the whole chain runs (about 1.5-2.5 h on the 8-core CPU container).

Stored columns (VERDICT r01 "cfg5 golden columns"; parity classes of SURVEY.md §8(c) P3):
  * j in {2000, 6000, 10000, 14000} +- 2: isolated at tau_v = 1e-6 ||T||_1, per-vector gate;
  * the top tau_v run [15948, 16000) (gaps <= tau_v): subspace gate.
The bottom run [0, 52) is cheap for the oracle's range mode and is recomputed by the test.
Also stored: the input w itself (the GPU test feeds this exact w, so the columns do not
depend on the LAPACK build that produced it), info, the iteration count of every vector,
and a hash of w.

Usage: OMP_NUM_THREADS=6 python tests/golden/make_cfg5_golden.py [--full-out PATH]
"""
import argparse
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from paper_1209_1910_b200 import workloads as W  # noqa: E402

SEED = 1
COLS = sorted(set(j + k for j in (2000, 6000, 10000, 14000) for k in range(-2, 3)) | set(range(15948, 16000)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--full-out", default=None, help="also save the whole Z (2 GB) here")
    a = ap.parse_args()
    d, e, w = W.problem("cfg5")
    t0 = time.time()
    Z, info, iters = O.eigvecs(d, e, w, seed=SEED, return_iters=True)
    dt = time.time() - t0
    print(f"oracle cfg5: info={info} {dt:.0f} s, iters hist {np.bincount(iters)}", flush=True)
    if a.full_out:
        np.save(a.full_out, Z)
    cols = np.array(COLS, dtype=np.int64)
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cfg5_oracle_cols.npz")
    np.savez(out, cols=cols, w=w, Z=np.ascontiguousarray(Z[:, cols]), info=np.int64(info),
             iters=iters.astype(np.int8), seed=np.int64(SEED), oracle_seconds=np.float64(dt),
             w_sha=np.bytes_(hashlib.sha256(np.ascontiguousarray(w).tobytes()).hexdigest()))
    print("wrote", out)


if __name__ == "__main__":
    main()
