"""One parity check of a (scaled) config against the oracle: a short GPU smoke for risky changes."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
from paper_1209_1910_b200 import workloads as W  # noqa: E402
from paper_1209_1910_b200.tinv import Tinv  # noqa: E402
from tests.helpers import EPS, parity_report  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("cases", nargs="+")   # cfg:n
args = ap.parse_args()
h = Tinv(0)
h.set_profiling(True)
for c in args.cases:
    cfg, n = (c.split(":") + [None])[:2]
    d, e, w = W.problem(cfg, int(n) if n else None)
    dev = torch.device("cuda:0")
    t0 = time.time()
    Z, rc = h.eigvecs(*(torch.tensor(a, dtype=torch.float64, device=dev) for a in (d, e, w)), seed=1)
    torch.cuda.synchronize()
    dt = time.time() - t0
    Zg = Z.cpu().numpy()
    nn = len(d)
    tn = O.tnorm(d, e)
    TZ = d[:, None] * Zg
    TZ[:-1] += e[:, None] * Zg[1:]
    TZ[1:] += e[:, None] * Zg[:-1]
    res = np.linalg.norm(TZ - Zg * w, axis=0).max() / (nn * EPS * tn)
    orth = np.abs(Zg.T @ Zg - np.eye(nn)).max() / (nn * EPS)
    msg = f"{cfg}:{nn} rc={rc} res={res:.3f} orth={orth:.3f} t={dt:.2f}s"
    if nn <= 2500:
        Zo, _ = O.eigvecs(d, e, w, seed=1)
        wv, ws, nv, ng = parity_report(w, tn, Zg, Zo)
        msg += f" vec={wv:.2e} sub={1 - ws:.2e}"
    print(msg, {k: round(v, 3) for k, v in h.stats()["cwy_phase_ms"].items()}, flush=True)
