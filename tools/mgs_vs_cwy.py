"""Paper Tables 3-8 analogue: device time of the classical MGS
reorthogonalisation (Alg. 1) and of the ordinary compact-WY sequence (§3.3.1) against the
reduced compact-WY sequence (§3.3.2, the method) on one B200, for a single eigen-cluster of m
vectors inside n = 2000 (the rest in small clusters), and on cfg1/cfg2 (resident kernel);
with --wide, the persistent kernel's regime m ~ n: the paper's Type 2 (all-ones, one cluster of
n) at n = 1050, 2100, 4200, and cfg4 at n = 2000, 4000 (and 8000 with --full).
Reps adapt to the run time (>= 1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1209_1910_b200 import workloads as W  # noqa: E402
from paper_1209_1910_b200.tinv import Tinv  # noqa: E402


def clustered(n, m, seed=3):
    rng = np.random.default_rng(seed)
    rest = n - m
    groups = [m] + [3] * (rest // 3) + ([rest % 3] if rest % 3 else [])
    rng.shuffle(groups)
    d = np.concatenate([g + 1e-7 * rng.uniform(-1, 1, k) for g, k in enumerate(groups)])
    e = 1e-9 * rng.uniform(-1, 1, n - 1)
    return d, e, W.eigenvalues(d, e)


def time_mode(h, prob, mode, reps=10):
    if "--wide" in sys.argv:
        reps = 1
    d, e, w = (torch.tensor(a, dtype=torch.float64, device="cuda:0") for a in prob)
    Z = torch.empty((len(d), len(d)), dtype=torch.float64, device="cuda:0")
    h.set_reorth(mode)
    for _ in range(1 if "--wide" in sys.argv else 3):
        h.eigvecs(d, e, w, Z=Z, seed=1)
    torch.cuda.synchronize()
    s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        _, rc = h.eigvecs(d, e, w, Z=Z, seed=1)
    t.record()
    torch.cuda.synchronize()
    assert rc == 0
    return s.elapsed_time(t) / reps


h = Tinv(0)
if "--wide" in sys.argv:
    cases = [(f"type2 n={n} (one cluster of n)", W.problem("type2", n)) for n in (1050, 2100, 4200)]
    cases += [(f"cfg4 n={n} (one cluster of n)", W.problem("cfg4", n)) for n in ((2000, 4000, 8000) if "--full" in sys.argv else (2000, 4000))]
else:
    cases = [("cfg1", W.problem("cfg1")), ("cfg2", W.problem("cfg2"))]
    cases += [(f"n=2000, one cluster m={m}", clustered(2000, m)) for m in (8, 16, 32, 48, 60)]
print("case, t_cwy ms (reduced, §3.3.2), t_ordinary ms (§3.3.1), t_mgs ms (Alg. 1), t_ordinary/t_cwy, t_mgs/t_cwy")
for name, prob in cases:
    tc = time_mode(h, prob, "cwy")
    to = time_mode(h, prob, "ordinary")
    tm = time_mode(h, prob, "mgs")
    print(f"{name}, {tc:.3f}, {to:.3f}, {tm:.3f}, {to / tc:.2f}, {tm / tc:.2f}", flush=True)
h.set_reorth("cwy")
