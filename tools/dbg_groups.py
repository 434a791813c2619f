"""Resident-group timeline of one config (TINV_DEBUG prints of the last call) and the mean
device time of a few calls.  Usage: python tools/dbg_groups.py cfg2 [calls]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1209_1910_b200 import workloads as W  # noqa: E402
from paper_1209_1910_b200.tinv import Tinv  # noqa: E402

cfg = sys.argv[1]
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 10
d, e, w = (torch.tensor(a, dtype=torch.float64, device="cuda:0") for a in W.problem(cfg))
h = Tinv(0)
Z = torch.empty((len(d), len(d)), dtype=torch.float64, device="cuda:0")
for _ in range(3):
    h.eigvecs(d, e, w, seed=1, Z=Z)
torch.cuda.synchronize()
s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(calls):
    h.eigvecs(d, e, w, seed=1, Z=Z)
t.record()
torch.cuda.synchronize()
print(f"{cfg} env={ {k: v for k, v in os.environ.items() if k.startswith('TINV_')} } {s.elapsed_time(t) / calls:.3f} ms/call", flush=True)
h.set_profiling(True)
os.environ["TINV_DEBUG"] = "1"
h.eigvecs(d, e, w, seed=1, Z=Z)
torch.cuda.synchronize()
del os.environ["TINV_DEBUG"]
st = h.stats()
print({k: round(v, 3) for k, v in st["kernel_ms"].items()}, flush=True)
