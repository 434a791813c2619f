"""Times cfg4 tinv_eigvecs calls under environment variants (knobs read per call): one
line per variant with the mean device time of 2 calls and the phase timers of a third."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1209_1910_b200 import workloads as W  # noqa: E402
from paper_1209_1910_b200.tinv import Tinv  # noqa: E402

cfg = sys.argv[1]
variants = sys.argv[2:]
d, e, w = W.problem(cfg, None)
dev = torch.device("cuda:0")
args = [torch.tensor(a, dtype=torch.float64, device=dev) for a in (d, e, w)]
h = Tinv(0)
h.eigvecs(*args, seed=1)
torch.cuda.synchronize()
for v in variants:
    env = dict(kv.split("=") for kv in v.split(",") if kv)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    ts = []
    for _ in range(2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        h.eigvecs(*args, seed=1)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    h.set_profiling(True)
    h.eigvecs(*args, seed=1)
    torch.cuda.synchronize()
    ph = h.stats()["cwy_phase_ms"]
    h.set_profiling(False)
    for k, o in old.items():
        if o is None:
            os.environ.pop(k)
        else:
            os.environ[k] = o
    print(f"{cfg} [{v}] {sum(ts)/len(ts):.1f} ms  " + " ".join(f"{k}={x:.0f}" for k, x in ph.items() if x), flush=True)
