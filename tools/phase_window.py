"""Per-phase cost of the wide compact-WY kernel for the vectors j_c in a window (TINV_PROF_P0/P1):
microseconds per iteration of each phase next to the rate its paper-sequence bytes imply.
Usage: python tools/phase_window.py cfg4 [p0:p1 ...]
The windows and TINV_PROF_CTA need a debug build: make -C paper_1209_1910_b200/csrc -B EXTRA=-DTINV_WIDE_DEBUG"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1209_1910_b200 import workloads as W  # noqa: E402
from paper_1209_1910_b200.tinv import Tinv  # noqa: E402

cfg = sys.argv[1]
wins = [tuple(int(x) for x in a.split(":")) for a in sys.argv[2:]] or [(500, 600), (3950, 4050), (7400, 7500)]
d, e, w = W.problem(cfg, int(os.environ["PW_N"]) if os.environ.get("PW_N") else None)
n = len(d)
dev = torch.device("cuda:0")
args = [torch.tensor(a, dtype=torch.float64, device=dev) for a in (d, e, w)]
h = Tinv(0)
h.set_profiling(True)
h.eigvecs(*args, seed=1)
torch.cuda.synchronize()
for p0, p1 in wins:
    os.environ["TINV_PROF_P0"], os.environ["TINV_PROF_P1"] = str(p0), str(p1)
    h.eigvecs(*args, seed=1)
    torch.cuda.synchronize()
    ph = h.stats()["cwy_phase_ms"]
    nv = p1 - p0
    its = 2 * nv
    p = 0.5 * (p0 + p1)
    by = {"A": 8 * (n * p - p * p / 2), "TT": 8 * p * p / 2, "BC": 16 * (n - p) * p, "TN": 8 * p * p / 2,
          "D": 8 * (n * p - p * p / 2)}
    row = []
    for k, v in ph.items():
        if v == 0:
            continue
        per = 1e3 * v / (nv if k in ("A", "solve_fwd", "solve_back", "solve_wait") else its)
        s = f"{k}={per:.1f}us"
        if k in by:
            s += f"({by[k] / per / 1e6:.2f}TB/s)"
        row.append(s)
    print(f"{cfg} n={n} p=[{p0},{p1}):", " ".join(row), flush=True)
