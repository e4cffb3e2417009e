"""Copies one round's GPU evidence from gpurun_out/ into profiles/ (tracked).

    python tools/summarize_profiles.py r01

  gpurun_out/bench_plain.json  -> profiles/<tag>_bench_line.json
  gpurun_out/launches.csv      -> profiles/<tag>_bench_launches_raw.csv (kernel, us)
                                  profiles/<tag>_bench_launches_summary.csv (per kernel)
  gpurun_out/<name>.ncu-rep    -> profiles/<tag>_<name>_summary.csv (selected metrics)
(the files tools/profile_round.sh writes on the GPU box).
"""
import collections
import csv
import io
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.environ.get("PROFILE_OUT", os.path.join(ROOT, "profiles"))
METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
    "launch__shared_mem_per_block_dynamic",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
]


def short(name: str) -> str:
    name = name.split("(")[0]
    for p in ("void ", "pp::"):
        if name.startswith(p):
            name = name[len(p):]
    return name.split("<")[0] if not name.startswith("at::") else name


def launches(tag: str, src_name: str = "launches.csv", out_name: str = "bench_launches") -> None:
    src = os.path.join(OUT, src_name)
    lines = [l for l in open(src) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    raw = [(r["Kernel Name"], float(r["Metric Value"]) / 1000.0) for r in rows
           if r["Metric Name"] == "gpu__time_duration.sum"]
    with open(os.path.join(PROF, f"{tag}_{out_name}_raw.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "us"])
        for k, us in raw:
            w.writerow([k, f"{us:.3f}"])
    agg = collections.defaultdict(list)
    for k, us in raw:
        agg["pp::" + short(k) if "pp::" in k else short(k)].append(us)
    total = sum(us for _, us in raw)
    with open(os.path.join(PROF, f"{tag}_{out_name}_summary.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "launches", "total_us", "mean_us", "share_of_profiled_time"])
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            w.writerow([k, len(v), f"{sum(v):.1f}", f"{sum(v) / len(v):.2f}", f"{sum(v) / total:.4f}"])


def ncu_summary(tag: str, name: str) -> None:
    rep = os.path.join(OUT, f"{name}.ncu-rep")
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    with open(os.path.join(PROF, f"{tag}_{name}_summary.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "metric", "unit", "value"])
        kernel = vals[hdr.index("Kernel Name")]
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                w.writerow([kernel, m, units[i], vals[i]])


def main() -> int:
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    shutil.copy(os.path.join(OUT, "bench_plain.json"), os.path.join(PROF, f"{tag}_bench_line.json"))
    launches(tag)
    if os.path.exists(os.path.join(OUT, "launches_mp1024.csv")):
        launches(tag, "launches_mp1024.csv", "minplus_c1024_launches")
    for name in sys.argv[2:] or ["mp_fold_full", "fused_full"]:
        ncu_summary(tag, name)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
