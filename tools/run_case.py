"""Run tinv_eigvecs once (after warm-up) on a named config -- a short target for ncu."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1209_1910_b200 import workloads as W  # noqa: E402
from paper_1209_1910_b200.tinv import Tinv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--profile", action="store_true")
args = ap.parse_args()
d, e, w = W.problem(args.config, args.n)
dev = torch.device("cuda:0")
dd, de, dw = (torch.tensor(x, dtype=torch.float64, device=dev) for x in (d, e, w))
h = Tinv(0)
h.set_profiling(args.profile)
for _ in range(args.reps):
    Z, rc = h.eigvecs(dd, de, dw, seed=1)
torch.cuda.synchronize()
st = h.stats()
print(args.config, len(d), "rc", rc, "kernel_ms", st["kernel_ms"], "phases", st["cwy_phase_ms"])
