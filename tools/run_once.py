"""One tinv_eigvecs call of a config on cuda:0 (for profiler captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1209_1910_b200 import workloads as W  # noqa: E402
from paper_1209_1910_b200.tinv import Tinv  # noqa: E402

d, e, w = W.problem(sys.argv[1], None)
args = [torch.tensor(a, dtype=torch.float64, device="cuda:0") for a in (d, e, w)]
h = Tinv(0)
Z, rc = h.eigvecs(*args, seed=1)
torch.cuda.synchronize()
print("rc", rc)
