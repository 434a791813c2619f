"""Summarise ncu outputs for profiles/: a launch list (--metrics gpu__time_duration.sum
--csv) aggregated per kernel, and the headline counters of `--set full` reports."""
import csv
import subprocess
import sys
from collections import defaultdict

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_membar",
        "smsp__pcsamp_warps_issue_stalled_wait", "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
        "smsp__pcsamp_warps_issue_stalled_short_scoreboard", "smsp__pcsamp_warps_issue_stalled_sleeping",
        "smsp__pcsamp_warps_issue_stalled_selected", "smsp__pcsamp_warps_issue_stalled_lg_throttle",
        "smsp__pcsamp_warps_issue_stalled_no_instructions", "smsp__pcsamp_sample_count"]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[1:]:
        agg[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    print(f"# launch list {path}: kernel, launches, mean us, share of all kernel time")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k}, {len(v)}, {sum(v) / len(v) / 1e3:.2f}, {sum(v) / tot:.4f}")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, units = r[0], r[1]
    print(f"# ncu --set full {path}")
    for v in r[2:]:
        print("kernel:", v[h.index("Kernel Name")])
        for w in WANT:
            if w in h:
                i = h.index(w)
                print(f"  {w} = {v[i]} {units[i]}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        (launches if p.endswith(".csv") else full)(p)
