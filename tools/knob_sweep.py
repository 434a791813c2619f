"""Time tinv_eigvecs on one config for several values of one environment knob (read per call),
in one process on one handle: python tools/knob_sweep.py --config cfg5 --knob TINV_CTA0 --values 0,60,100"""
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
ap.add_argument("--knob", required=True)
ap.add_argument("--values", required=True)
ap.add_argument("--sep", default=",", help="separator of --values (for values that contain commas)")
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--rounds", type=int, default=1, help="repeat the whole value list (drift check)")
args = ap.parse_args()
d, e, w = W.problem(args.config, args.n)
dev = torch.device("cuda:0")
dd, de, dw = (torch.tensor(x, dtype=torch.float64, device=dev) for x in (d, e, w))
h = Tinv(0)
h.set_profiling(True)
Z, rc = h.eigvecs(dd, de, dw, seed=1)   # allocation + warm-up
keys = ("first", "TT", "BC", "TN", "D", "solve_back", "solve_wait")
kms = ("batched_lu", "cwy")
for rnd in range(args.rounds):
    for v in args.values.split(args.sep):
        os.environ[args.knob] = v
        ts = []
        for _ in range(args.reps):
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record()
            Z, rc = h.eigvecs(dd, de, dw, seed=1)
            t1.record()
            torch.cuda.synchronize()
            ts.append(t0.elapsed_time(t1))
        st = h.stats()
        ph = st["cwy_phase_ms"]
        print(f"{args.config} n={len(d)} {args.knob}={v} rc={rc} ms={min(ts):.3f} " +
              " ".join(f"{k}_ms={st['kernel_ms'][k]:.3f}" for k in kms) + " " +
              " ".join(f"{k}={ph[k]:.1f}" for k in keys if k in ph), flush=True)
