#!/usr/bin/env python
"""Benchmark of the hot path: all n eigenvectors of a symmetric tridiagonal T by inverse
iteration with compact-WY reorthogonalisation (DSTEIN-cWY, Alg. 4), fp64.

Metric (BASELINE.json): eigenvectors/s (all n, fp64) at n = 2000-16000; reorth HBM GB/s vs
peak.  One step = one tinv_eigvecs call on one synthetic input resident in HBM.  Default
workload: configs[4] (cfg5, n = 16000, the top of the metric's n range; one cluster of 16000
vectors): the HBM-bound regime the metric's "reorth HBM GB/s vs peak" half refers to, ~18 s
per step.  Other configs: --config cfg1..cfg5 (cfg4 = n = 8000, one cluster; cfg2 = the
n = 2000 many-small-clusters, latency-bound case).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg5] [--impl tinv|reference]

--gpus N > 1 without a torch.distributed environment re-executes itself under
torch.distributed.run (one process per GPU, NCCL, 127.0.0.1).  Multi-rank: a single giant
cluster (cfg4, cfg5) is row-split over the ranks (in-kernel reductions over NVLink peer
memory); otherwise the clusters are sharded by columns and each rank's columns broadcast at
the end.  Either way the whole job computes one problem (strong scaling).
The timed Z is checked on the device after the timed region (P0 invariants of
BASELINE.json north_star); a violation prints the line with "parity.ok": false and exits 1.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1209_1910_b200 import workloads as W  # noqa: E402

WORKLOAD_DESC = {
    "cfg1": "n=200 1D Laplacian (configs[0])",
    "cfg2": "n=2000 random tridiagonal d,e~U(-1,1), seed 0 (configs[1])",
    "cfg3": "n=4200 glued Wilkinson W21+ x200, glue 1e-10 (configs[2])",
    "cfg4": "n=8000 single giant cluster d=1+1e-7U, e=1e-9U (configs[3])",
    "cfg5": "n=16000 perturbed Laplacian 2+1e-6U(-1,1), -1 (configs[4])",
}


BIG = ("cfg4", "cfg5")          # one giant cluster: row split at N > 1, seconds per step
FP64_DFMA_TFLOPS = 36.5     # measured fp64 DFMA rate of this B200 (tools/micro/fp64_peak.cu)


def config_dict(args, n, ws):
    """The workload description -- identical in both arms (no run-dependent keys)."""
    par = "single GPU" if ws == 1 else (f"row-split x{ws}" if args.config in BIG else f"cluster-shard x{ws}")
    return {"workload": WORKLOAD_DESC[args.config], "name": args.config, "n": n, "parallelism": par,
            "reorth": args.reorth, "l2": "flushed between timed steps (256 MB write)", "seed": args.seed}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


class ClockSampler:
    """SM clocks and throttle reasons sampled every 20 ms during the timed region (NVML)."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        try:
            import pynvml as N

            N.nvmlInit()
            hdl = N.nvmlDeviceGetHandleByIndex(self.index)
            mx = N.nvmlDeviceGetMaxClockInfo(hdl, N.NVML_CLOCK_SM)
            bits = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                    "sw_power_cap": 0x4}
            while not self._stop.is_set():
                sm = N.nvmlDeviceGetClockInfo(hdl, N.NVML_CLOCK_SM)
                rs = N.nvmlDeviceGetCurrentClocksEventReasons(hdl)
                self.samples.append((sm, mx, [k for k, b in bits.items() if rs & b]))
                self._stop.wait(0.02)
        except Exception as exc:  # pragma: no cover
            self.samples.append((None, None, [f"nvml error: {exc}"]))

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.05)
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        sm = [s[0] for s in self.samples if s[0] is not None]
        mx = [s[1] for s in self.samples if s[1] is not None]
        reasons = sorted({r for s in self.samples for r in s[2]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def reference_arm(args):
    """--impl reference: the CPU oracle as it stands, on this arm's config/metric."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    if ws > 1:   # torchrun sets OMP_NUM_THREADS=1 per rank; rank 0 alone works here: all host cores
        os.environ["OMP_NUM_THREADS"] = str(os.cpu_count() or 1)
    import oracle as O

    d, e, w = W.problem(args.config)
    n = len(d)
    # a bounded sample per step: the full problem when it takes seconds, else the first
    # vectors of the spectrum (whole clusters from their start), sized to ~10 s
    full = n <= 4200
    j_hi = n if full else {"cfg4": 256, "cfg5": 160}.get(args.config, 256)
    for _ in range(args.warmup if full else 0):
        O.eigvecs(d, e, w, seed=1, j_lo=0, j_hi=j_hi)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.eigvecs(d, e, w, seed=1, j_lo=0, j_hi=j_hi)
    dt = (time.perf_counter() - t0) / args.steps
    value = j_hi / dt
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    sample = "all n eigenvectors" if full else f"first {j_hi} of {n} eigenvectors (one cluster, from its start)"
    line = {
        "impl": "reference", "metric": "eigenvectors/s (all n, fp64)", "value": value, "unit": "eigenvectors/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args, n, ws),
        "cpu_baseline": {"value": value, "unit": "eigenvectors/s", "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "eigenvectors/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def cpu_baseline(d, e, w, budget_s=12.0, mgs=False):
    """The oracle timed on this host's cores on a bounded sample of the workload."""
    import oracle as O

    n = len(d)
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    t0 = time.perf_counter()
    if n <= 4200:
        reps = 0
        while True:
            O.eigvecs(d, e, w, seed=1, mgs=mgs)
            reps += 1
            if time.perf_counter() - t0 > budget_s or reps >= 50:
                break
        dt = time.perf_counter() - t0
        return {"value": n * reps / dt, "unit": "eigenvectors/s", "cores": cores, "kind": "oracle",
                "sample": f"{reps} full run(s) of all {n} eigenvectors, {dt:.1f} s"}
    k = 160 if n > 10000 else 256
    O.eigvecs(d, e, w, seed=1, j_lo=0, j_hi=k, mgs=mgs)
    dt = time.perf_counter() - t0
    return {"value": k / dt, "unit": "eigenvectors/s", "cores": cores, "kind": "oracle",
            "sample": f"first {k} of {n} eigenvectors (start of the single cluster; later vectors cost more), {dt:.1f} s"}


def p0_check(torch, d, e, w, Zt, dev):
    """P0 invariants (BASELINE.json north_star) of the timed result, on the device:
    max_j ||T z_j - w_j z_j||_2 <= 10 n eps ||T||_1 and max |Z^T Z - I| <= 10 n eps.
    Zt's row j is eigenvector j (column-major Z).  fp64 throughout (cuBLAS DGEMM for Z^T Z)."""
    n = len(d)
    eps = 2.0 ** -53
    dt, wt = (torch.tensor(a, dtype=torch.float64, device=dev) for a in (d, w))
    TZ = Zt * dt[None, :]
    if n > 1:
        et = torch.tensor(e, dtype=torch.float64, device=dev)
        TZ[:, :-1] += Zt[:, 1:] * et[None, :]
        TZ[:, 1:] += Zt[:, :-1] * et[None, :]
    TZ -= Zt * wt[:, None]
    tn = float(np.max(np.abs(d) + np.concatenate([[0.0], np.abs(e)]) + np.concatenate([np.abs(e), [0.0]])))
    res = torch.linalg.vector_norm(TZ, dim=1).max().item() / (n * eps * tn)
    del TZ
    G = Zt @ Zt.t()
    G.diagonal().sub_(1.0)
    orth = G.abs().max().item() / (n * eps)
    del G
    ok = bool(res <= 10.0 and orth <= 10.0)
    return {"ok": ok, "residual_n_eps_tnorm": res, "orth_n_eps": orth, "bound": 10.0,
            "what": "P0 invariants of the last timed step's Z, on the device"}


def e2e_leg(h, d, e, w, n, args, ws, dev, barrier):
    """The same metric through tinv_eigvecs_host with pinned host buffers: H2D of d, e, w and
    the columns of Z landing in host memory inside the timed region."""
    import torch
    import torch.distributed as dist

    hd, he, hw = (torch.tensor(a, dtype=torch.float64).pin_memory() for a in (d, e, w))
    hZ = torch.empty((n, n), dtype=torch.float64).pin_memory()
    h.eigvecs_host(hd, he, hw, Z=hZ, seed=args.seed)
    barrier()
    e_steps = max(1, min(args.steps, 2 if args.config in BIG else 5))
    t0 = time.perf_counter()
    for _ in range(e_steps):
        h.eigvecs_host(hd, he, hw, Z=hZ, seed=args.seed)
    barrier()
    e_ms = (time.perf_counter() - t0) * 1e3 / e_steps
    if ws > 1:
        t = torch.tensor([e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t.item())
    e2e = {"value": n / (e_ms * 1e-3), "unit": "eigenvectors/s", "ms_per_step": e_ms,
           "h2d_bytes_per_step": 8 * (3 * n - 1), "d2h_bytes_per_step": 8 * n * n,
           "l2": "not flushed between e2e calls (back to back, as a user calls it)"}
    return e2e


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="timed steps (default 5 for cfg4/cfg5, else 30)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg5", choices=list(WORKLOAD_DESC))
    ap.add_argument("--impl", default="tinv", choices=["tinv", "reference"])
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer leg (profiler runs)")
    ap.add_argument("--reorth", default="cwy", choices=["cwy", "mgs", "ordinary"],
                    help="cwy: compact WY (Alg. 4, reduced §3.3.2 sequence, the method); mgs: classical MGS "
                         "(Alg. 1), the paper's comparison; ordinary: compact WY in the §3.3.1 sequence")
    ap.add_argument("--verbose", action="store_true")
    args = ap.parse_args()
    if args.steps is None:
        args.steps = 5 if args.config in BIG else 30
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # honour --gpus N: one process per GPU under torch.distributed.run (127.0.0.1)
        import socket
        import subprocess

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    ws_env = int(os.environ.get("WORLD_SIZE", "1"))
    if ws_env != args.gpus:
        print(f"bench.py: WORLD_SIZE={ws_env} but --gpus {args.gpus}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return reference_arm(args)
    args.warmup = max(args.warmup, 3)

    import torch
    import torch.distributed as dist

    from paper_1209_1910_b200.tinv import Tinv

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    nccl_id = None
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
        # the library's own communicator: rank 0 makes the id, torch.distributed ships it
        import ctypes as C

        buf = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            lib = C.CDLL("libnccl.so.2", mode=C.RTLD_GLOBAL)
            uid = (C.c_char * 128)()
            assert lib.ncclGetUniqueId(uid) == 0
            buf = torch.frombuffer(bytearray(uid.raw), dtype=torch.uint8).clone()
        obj = [buf.numpy().tobytes()]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]

    d, e, w = W.problem(args.config)
    n = len(d)
    dd, de, dw = (torch.tensor(a, dtype=torch.float64, device=dev) for a in (d, e, w))
    Zt = torch.empty((n, n), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    h = Tinv(local, stream=stream, nranks=ws, rank=rank, nccl_id=nccl_id)
    h.set_reorth(args.reorth)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)   # > 126 MB L2

    def barrier():
        torch.cuda.synchronize(dev)
        if ws > 1:
            dist.barrier()

    for _ in range(args.warmup):
        h.eigvecs(dd, de, dw, Z=Zt, seed=args.seed)
    barrier()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    kms = {}
    launches = 0
    rcs = []
    with ClockSampler(local) as clk:
        barrier()
        for k in range(args.steps):
            flush.fill_(float(k))                     # L2 flush between timed steps (untimed)
            ev[k][0].record(stream)
            _, rc = h.eigvecs(dd, de, dw, Z=Zt, seed=args.seed)
            ev[k][1].record(stream)
            rcs.append(rc)
            launches += h.stats()["launches"]
        barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    parity = p0_check(torch, d, e, w, Zt, dev)     # the Z of the last timed step (untimed)
    # per-kernel breakdown and phase timers from separate profiled calls (the library's events
    # and host synchronisation would otherwise sit inside the timed steps)
    h.set_profiling(True)
    for k in range(min(1 if args.config in BIG else 3, args.steps)):
        flush.fill_(float(k))
        h.eigvecs(dd, de, dw, Z=Zt, seed=args.seed)
        stp = h.stats()
        for kk, v in stp["kernel_ms"].items():
            kms.setdefault(kk, []).append(v)
        kms.setdefault("dz", []).append(stp["dz_ms"])
    h.set_profiling(False)
    barrier()
    tot_ms = float(sum(step_ms))
    if ws > 1:
        t = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    ms_per_step = tot_ms / args.steps
    value = n / (ms_per_step * 1e-3)
    st = h.stats()

    # ---- roofline of the dominant kernel (library events on the launching stream)
    peaks, src = measured_peaks()
    avg = {k: float(np.mean(v)) for k, v in kms.items() if k != "total"}
    dom = max(("batched_lu", "cwy"), key=lambda k: avg.get(k, 0.0))
    if dom == "cwy":
        alg_bytes = st["reorth_bytes"]
    else:
        alg_bytes = st["solve_bytes"]
    achieved = alg_bytes / (avg[dom] * 1e-3) / 1e9 if avg.get(dom, 0) > 0 else 0.0
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tr = json.load(f).get(args.config)
        if tr and tr.get("kernel") == dom:
            traffic = float(tr["bytes"])
    except Exception:
        traffic = None
    resident = dom == "cwy" and st.get("resident_groups", 0) > 0
    kernel_name = {"cwy": "cwy_resident_kernel" if resident else "cwy_kernel (persistent, wide clusters)",
                   "batched_lu": "batched_lu_kernel"}[dom]
    roof = {"kernel": kernel_name, "bound": "latency" if resident else "hbm", "achieved": achieved,
            "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
            "peak_source": src, "alg_bytes_per_launch": alg_bytes, "kernel_ms": avg[dom],
            "share_of_step": avg[dom] / ms_per_step if ms_per_step > 0 else None}
    if traffic:
        # measured DRAM bytes of the same kernel (committed ncu capture) over the same kernel time
        roof["traffic_gbs"] = traffic / (avg[dom] * 1e-3) / 1e9
        roof["traffic_frac"] = roof["traffic_gbs"] / peaks["hbm_gbs"]
    if dom == "cwy" and not resident and st.get("dz_parked", 0) > 0:
        # the deferred final pass D: its GEMM runs after the persistent kernel
        # inside the same cWY interval, so the cWY bytes are over both; the GEMM itself is an fp64
        # DFMA contraction reported against the measured DFMA peak
        roof["kernel"] = "cwy_kernel + dz_gemm_kernel/dz_finish_kernel (deferred final pass D)"
        dzms = avg.get("dz", 0.0)
        roof["dz"] = {"kernel": "dz_gemm_kernel + dz_finish_kernel", "parked": st["dz_parked"], "ms": dzms,
                      "share_of_step": dzms / ms_per_step if ms_per_step > 0 else None}
        if st["nclusters"] == 1 and st["dz_parked"] == n - 64 and dzms > 0:
            p = np.arange(64, n, dtype=np.float64)
            flops = float(np.sum(2.0 * ((p + 1) * (p + 2) / 2 + (n - p - 1) * (p + 1))))
            roof["dz"].update({"bound": "alu", "flops": flops, "achieved": flops / (dzms * 1e-3) / 1e12,
                               "peak": FP64_DFMA_TFLOPS, "unit": "TFLOP/s",
                               "frac": flops / (dzms * 1e-3) / 1e12 / FP64_DFMA_TFLOPS,
                               "peak_source": "measured DFMA rate, tools/micro/fp64_peak.cu (DESIGN.md section 8)"})
    if resident:
        roof["note"] = ("resident cWY kernel: Y stays in shared memory, so DRAM traffic is far below the "
                        "algorithmic bytes; the step is bound by the dependent chains and phase latencies "
                        "(DESIGN.md section 8), not by HBM: 'frac' is the algorithmic-byte rate over the HBM peak")

    # ---- e2e through the public API with host buffers (pinned)
    if args.no_e2e:
        e2e = None
    else:
        e2e = e2e_leg(h, d, e, w, n, args, ws, dev, barrier)

    line = {
        "metric": "eigenvectors/s (all n, fp64)", "value": value, "unit": "eigenvectors/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args, n, ws),
        "roofline": roof,
        "parity": parity,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "info": {"return_codes": sorted(set(rcs)), "nclusters": st["nclusters"], "max_cluster": st["max_cluster"],
                 "n_clustered": st["n_clustered"], "iters_hist": st["iters_hist"], "kernel_ms": avg,
                 "cwy_phase_ms": st["cwy_phase_ms"], "group_syncs": st["group_syncs"], "ngroups": st["ngroups"],
                 "cwy_ctas": st["cwy_ctas"], "dz_parked": st["dz_parked"], "dz_redo": st["dz_redo"],
                 "step_ms_min": min(step_ms), "step_ms_max": max(step_ms)},
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(d, e, w, mgs=args.reorth == "mgs")
    ok = parity["ok"]
    if ws > 1:
        t = torch.tensor([0.0 if ok else 1.0], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ok = t.item() == 0.0
    if rank == 0:
        print(json.dumps(line))
        if not ok:
            print("bench.py: PARITY FAILURE (P0 invariants violated on the timed Z)", file=sys.stderr)
    h.close()
    if ws > 1:
        dist.destroy_process_group()
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
