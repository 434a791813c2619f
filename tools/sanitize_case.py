"""One small tinv_eigvecs call for compute-sanitizer runs (memcheck / racecheck / synccheck /
initcheck).  Usage: python tools/sanitize_case.py CASE  with CASE in
cfg1 | cfg2 | cfg4s (cfg4 family, n = 600) | vr2 (cfg4 n = 600 row split over 2 virtual ranks)
| cfg3s (glued W21+, n = 630) | mgs (cfg2 n = 800, MGS mode).
Checks the P0 invariants on the result (no oracle needed) and exits non-zero on failure."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1209_1910_b200 import workloads as W  # noqa: E402
from paper_1209_1910_b200.tinv import Tinv  # noqa: E402

case = sys.argv[1]
cfg, n = {"cfg1": ("cfg1", None), "cfg2": ("cfg2", None), "cfg4s": ("cfg4", 600), "vr2": ("cfg4", 600),
          "cfg3s": ("cfg3", 630), "mgs": ("cfg2", 800), "cfg5s": ("cfg5", 1500)}[case]
d, e, w = W.problem(cfg, n)
n = len(d)
h = Tinv(0)
if case == "vr2":
    h.set_virtual_ranks(2)
if case == "mgs":
    h.set_reorth("mgs")
dev = torch.device("cuda:0")
Z, rc = h.eigvecs(*(torch.tensor(a, dtype=torch.float64, device=dev) for a in (d, e, w)), seed=1)
torch.cuda.synchronize()
Zh = Z.cpu().numpy()
T = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
eps = 2.0 ** -53
tn = np.abs(T).sum(0).max()
res = np.linalg.norm(T @ Zh - Zh * w, axis=0).max() / (n * eps * tn)
orth = np.abs(Zh.T @ Zh - np.eye(n)).max() / (n * eps)
st = h.stats()
h.close()
print(f"{case}: n={n} rc={rc} residual={res:.3f} orth={orth:.3f} (x n eps) ngroups={st['ngroups']} "
      f"resident_groups={st['resident_groups']}")
sys.exit(0 if (rc == 0 and res <= 10 and orth <= 10) else 1)
