"""Back-sweep cycles per row of the resident kernel's unit 0 (TINV_RES_FLAGS=2 reports the
sweep's SM cycles in phase slot 15) for cfg2 and for a lone 25-vector cluster."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
from paper_1209_1910_b200 import workloads as W  # noqa: E402
from paper_1209_1910_b200.tinv import Tinv  # noqa: E402

os.environ["TINV_RES_FLAGS"] = "2"


def lone(n=2000, m=25, seed=3):
    rng = np.random.default_rng(seed)
    rest = n - m   # fillers of 3 keep fewer than ~900 groups 1e-3 ||T||_1 apart
    groups = [m] + [3] * (rest // 3) + ([rest % 3] if rest % 3 else [])
    d = np.concatenate([g * 1.0 + 1e-7 * rng.uniform(-1, 1, k) for g, k in enumerate(groups)])
    e = 1e-9 * rng.uniform(-1, 1, n - 1)
    return d, e, W.eigenvalues(d, e)


h = Tinv(0)
h.set_profiling(True)
for name, prob in (("cfg2", W.problem("cfg2")), ("lone25", lone())):
    d, e, w = (torch.tensor(a, dtype=torch.float64, device="cuda:0") for a in prob)
    for _ in range(3):
        Z, rc = h.eigvecs(d, e, w, seed=1)
    torch.cuda.synchronize()
    st = h.stats()
    ph = st["cwy_phase_ms"]
    cyc = ph["st_blkend"] * 1e6
    n = len(prob[0])
    print(f"{name}: rc={rc} sweep cycles total {cyc:.0f} -> per row per sweep (24 sweeps) {cyc / 24 / n:.2f}; back-sweep wall {ph['st_sync']:.3f} ms")
