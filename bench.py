#!/usr/bin/env python
"""bench.py — the driver's benchmark contract for the B200 planner.

Headline (BASELINE.json metric "Inception-v3 optimal-config search ms; min-plus
cell-updates/s vs FP32 roofline"), workload = BASELINE configs[2]:
``plan(inception_chain(batch=32, modules=12), DeviceGraph::uniform(16))`` —
the reference's Inception-v3 stand-in (109 layers, 144 edges) on 16 modelled
devices: cost tables (K1/K2) + node/edge-elimination DP to a 2-node graph
(K3/K4) + final enumeration (K5) + unwind, i.e. the paper's "~100 ms search".

* value      device ms per search, inputs resident in HBM: a prepared plan
             (one CUDA graph) launched K times, each bracketed by CUDA events
             on the planner's stream, L2 flushed (256 MiB write) between steps;
             N ranks each search their own replica -> whole-job ms per search
             = max-rank device time / (K*N)  (scaling "weak")
* e2e        the same search through the C ABI a user calls (pp_plan with host
             arrays): host prep + H2D of the descriptor image + device work +
             D2H of indices/cost, wall clock per call
* roofline   the min-plus fold kernel (K3) on the config-5 synthetic graph
             (1000 layers, bp 0.3, C configs per layer, exact int32 fixed
             point): achieved = 2 ops/cell x cells / wave-kernel time vs the
             FP32 CUDA-core peak 148 SM x 128 lanes x 2 x f_clk(measured)
* cpu_baseline  the real reference (oracle/_ref, compiled from
             /root/reference) plan() on the same workload, 1 host core

--impl reference runs the reference's CPU plan() on the same workload and
prints the same line with "impl": "reference".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
os.environ.setdefault("NCCL_DEBUG", "WARN")  # keep stdout to the one JSON line

METRIC = "Inception-v3 optimal-config search ms; min-plus cell-updates/s vs FP32 roofline"
PAPER_MS = 100.0  # PAPER.md:80 "about 100 ms" for Inception-v3 (120 nodes) on 16 GPUs


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "_fallback": True}


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def workload(name: str):
    """-> (model, batch, devices) ; synthetic handled separately."""
    if name.startswith("inception_chain@"):
        return "inception_chain", 32, int(name.split("@")[1])
    model, D = name.split("@")
    return model, 32, int(D)


# ---------------------------------------------------------------------------
# reference (CPU) arm
# ---------------------------------------------------------------------------

def reference_plan_ms(model, batch, D, runs, warmup=0):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    kind = "reference" if O.available("reference") else "port"
    g = O.Instance.builtin(model, batch, kind)
    times = []
    res = None
    for k in range(warmup + runs):
        t0 = time.perf_counter()
        g.build_tables(D)  # plan() = build_cost_tables + plan_with_tables (planner.hpp:368-371)
        res = g.plan()
        dt = (time.perf_counter() - t0) * 1e3
        if k >= warmup:
            times.append(dt)
    return kind, times, res


def _parallel_worker(spec):
    model, batch, D, barrier = spec
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    g = O.Instance.builtin(model, batch, "reference" if O.available("reference") else "port")
    barrier.wait()
    t0 = time.time()
    g.build_tables(D)
    g.plan()
    return t0, time.time()


def reference_parallel_ms(model, batch, D, procs, start="fork"):
    """Wall time of `procs` concurrent single-threaded plan() calls (one
    process per host core) / procs: the reference's throughput with every
    core busy, for comparison with the single-plan latency reported as the
    value (the reference's plan() itself cannot use more than one thread)."""
    import multiprocessing as mp

    ctx = mp.get_context(start)  # "spawn" from a process that has initialised CUDA
    with ctx.Manager() as m:
        barrier = m.Barrier(procs)
        with ctx.Pool(procs) as pool:
            spans = pool.map(_parallel_worker, [(model, batch, D, barrier)] * procs)
    return (max(e for _, e in spans) - min(s for s, _ in spans)) * 1e3 / procs


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    model, batch, D = workload(args.workload)
    kind, times, res = reference_plan_ms(model, batch, D, args.steps, args.warmup)
    v = statistics.mean(times)
    procs = os.cpu_count() or 1
    try:
        par = reference_parallel_ms(model, batch, D, procs)
    except Exception as exc:  # the latency line stands without it
        par = None
        print(f"parallel reference sample failed: {exc}", file=sys.stderr)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "ms", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": v, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": v / PAPER_MS, "dtype": "f64", "data": "synthetic (builtin model, analytic tables)",
        "config": {"workload": f"plan(inception_chain(12)@{D})" if model == "inception_chain" else args.workload,
                   "model": model, "batch": batch, "devices": D},
        "cpu_baseline": {"value": v, "unit": "ms", "cores": 1, "kind": kind,
                         "sample": f"{args.steps} full plan() calls (tables + DP) on 1 host core, single-threaded "
                                   f"reference compiled -O3 -DNDEBUG; nproc={os.cpu_count()}",
                         "all_cores_amortized_ms": par,
                         "all_cores_sample": f"{procs} concurrent plan() calls, one process per host core; "
                                             f"wall time / {procs} (throughput, not the latency above)"},
        "e2e": {"value": v, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "result": {"cost": res.cost, "node_eliminations": res.node_eliminations,
                   "edge_eliminations": res.edge_eliminations},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1802_04924_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    stream = torch.cuda.Stream()  # planner and timing events share this stream
    torch.cuda.set_stream(stream)
    ctx = P.Context(local, stream=stream.cuda_stream)
    model, batch, D = workload(args.workload)
    g = P.builtin_model(model if model != "inception_chain" else "inception_chain", batch)
    dev = P.DeviceGraph.uniform(D)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- value: prepared plan, device time per search --------------------------
    prep = P.PreparedPlan(g, devices=dev, ctx=ctx)
    for _ in range(args.warmup):
        flush.zero_()
        prep.launch()
        r = prep.fetch()
    launches0 = ctx.launches
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    barrier()
    with Clocks(local) as clk:
        for k in range(args.steps):
            flush.zero_()
            starts[k].record(stream)
            prep.launch()
            ends[k].record(stream)
        barrier()
    launches = ctx.launches - launches0
    r = prep.fetch()
    dev_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total = torch.tensor([sum(dev_ms)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(total, op=dist.ReduceOp.MAX)
    value = total.item() / (args.steps * world)

    # ---- e2e: pp_plan through the C ABI with host buffers ------------------------
    e2e = []
    h2d = d2h = 0
    for k in range(args.warmup + args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = P.plan(g, dev, ctx=ctx)
        dt = (time.perf_counter() - t0) * 1e3
        if k >= args.warmup:
            e2e.append(dt)
        h2d, d2h = res.h2d_bytes, res.d2h_bytes
    e2e_t = torch.tensor([sum(e2e)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_ms = e2e_t.item() / (args.steps * world)
    assert list(res.indices) == list(r.indices) and res.cost == r.cost

    # ---- per-kernel breakdown of the search -----------------------------------------
    prof = prep.profile()
    kern = {}
    for kind, ms, work in prof:
        k = kern.setdefault(kind, {"launches": 0, "ms": 0.0, "work": 0.0})
        k["launches"] += 1
        k["ms"] += ms
        k["work"] += work
    search_total = sum(v["ms"] for v in kern.values()) or 1.0
    for v in kern.values():
        v["share"] = v["ms"] / search_total

    # ---- plan_with_tables only (the CLI's planning_ms) ---------------------------------
    t_built = P.build_cost_tables(g, dev, ctx)
    pwt = P.PreparedPlan(g, tables=t_built, ctx=ctx)
    pw = []
    for k in range(args.warmup + args.steps):
        flush.zero_()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        pwt.launch()
        s1.record(stream)
        pwt.fetch()
        if k >= args.warmup:
            pw.append(s0.elapsed_time(s1))

    line = {
        "metric": METRIC, "value": value, "unit": "ms", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": max(dev_ms) if world == 1 else value * world, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": value / PAPER_MS, "dtype": "f64",
        "data": "synthetic (builtin model graph, analytic cost tables; each rank searches its own replica)",
        "config": {"workload": f"plan(inception_chain(12)@{D})" if model == "inception_chain" else args.workload,
                   "model": model, "batch": batch, "devices": D, "layers": g.n_layers, "edges": g.n_edges,
                   "l2": "256 MiB write between timed steps", "parallelism": f"replicas x{world}"},
        "e2e": {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "call": "pp_plan(ctx, graph, device_desc, k_bound, host indices) — host prep + H2D + device + D2H"},
        "gpu_launches": launches,
        "plan_with_tables_ms": statistics.mean(pw),
        "result": {"cost": r.cost, "node_eliminations": r.node_eliminations, "edge_eliminations": r.edge_eliminations,
                   "waves": r.waves, "precision": r.precision},
        "search_kernels": kern,
        "clocks": clk.summary(),
    }

    # ---- min-plus roofline (config-5 synthetic graph) --------------------------------
    if args.minplus_c > 0:
        line.update(minplus(P, ctx, args, flush, stream))

    # ---- CPU baseline: the real reference on the same workload --------------------------
    if rank == 0 and world == 1 and not args.no_cpu:
        kind, times, res_ref = reference_plan_ms(model, batch, D, args.cpu_runs)
        line["cpu_baseline"] = {
            "value": statistics.median(times), "unit": "ms", "cores": 1, "kind": kind,
            "sample": f"{args.cpu_runs} full plan() calls on {args.workload} (reference is single-threaded; "
                      f"nproc={os.cpu_count()})"}
        try:
            procs = os.cpu_count() or 1
            line["cpu_baseline"]["all_cores_amortized_ms"] = reference_parallel_ms(model, batch, D, procs, "spawn")
            line["cpu_baseline"]["all_cores_sample"] = (f"{procs} concurrent plan() calls, one process per host "
                                                        f"core; wall time / {procs} (throughput, not the latency)")
        except Exception as exc:
            print(f"parallel reference sample failed: {exc}", file=sys.stderr)
        line["result"]["matches_reference"] = bool(
            list(res_ref.indices) == list(r.indices) and res_ref.cost == r.cost)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def committed_traffic(kernel):
    """DRAM bytes (read + write) of one launch of `kernel` from the committed
    ncu --set full summary under profiles/ (the roofline's traffic field)."""
    import csv
    import glob

    for path in sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r*_full_summary.csv")),
                       reverse=True):
        with open(path) as f:
            rows = [r for r in csv.DictReader(f) if kernel in r["kernel"]]
        if not rows:
            continue
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        total = 0.0
        for r in rows:
            if r["metric"] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                total += float(r["value"]) * scale.get(r["unit"], 1.0)
        return total, f"{os.path.basename(path)}: dram__bytes_read.sum + dram__bytes_write.sum of one captured launch"
    return None, "no committed ncu --set full summary"


def minplus(P, ctx, args, flush, stream):
    """Config-5 synthetic sweep point: 1000 layers (bp 0.3, seed 1 topology),
    C configs per layer, device-generated dyadic tables, exact int32 DP."""
    import torch

    C = args.minplus_c
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:  # one plan row-sharded across all ranks (NCCL all-gathers at re-association points)
        from paper_1802_04924_b200 import distributed as PD

        ctx = P.Context(ctx.device, stream=stream.cuda_stream)
        PD.attach(ctx)
    g = P.series_parallel_graph(1, 1000, 0.3)
    t = P.synthetic_cost_tables(g, C, seed=1, ctx=ctx)
    prep = P.PreparedPlan(g, tables=t, ctx=ctx)
    prep.launch()
    r = prep.fetch()
    global_cells = float(C) ** 3 * sum(1 for rec in g.schedule()[0] if rec[0] == 0)
    with Clocks(ctx.device) as clk:
        runs = [prep.profile() for _ in range(args.minplus_runs)]
    # whole-plan device time of one search, max over ranks
    starts, ends = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    starts.record(stream)
    prep.launch()
    ends.record(stream)
    prep.fetch()
    plan_ms = starts.elapsed_time(ends)
    if world > 1:
        from paper_1802_04924_b200 import distributed as PD

        plan_ms = PD.max_over_ranks(plan_ms, device="cuda")
    folds = [(ms, w) for run in runs for kind, ms, w in run if kind == "mp_fold"]
    if not folds:  # generic path only (no certified large folds)
        folds = [(ms, w) for run in runs for kind, ms, w in run if kind == "wave"]
    wave_ms = sum(ms for ms, _ in folds) / len(runs)
    cells = sum(w for _, w in folds) / len(runs)
    total_ms = sum(ms for run in runs for _, ms, _ in run) / len(runs)
    by_kind = {}
    for run in runs:
        for kind, ms, _ in run:
            by_kind[kind] = by_kind.get(kind, 0.0) + ms / len(runs)
    c = clk.summary()
    pk = peaks()
    f_mhz = c["sm_mhz"] or pk.get("sm_max_mhz", 1965.0)
    sms = 148
    peak_tflops = sms * 128 * 2 * f_mhz * 1e6 / 1e12  # FP32 CUDA-core: 2 ops (add + min) per cell at 1 cell/lane/clk
    achieved = 2.0 * cells / (wave_ms * 1e-3) / 1e12
    traffic, traffic_basis = committed_traffic("mp_fold_kernel")
    return {
        "roofline": {"bound": "fp32", "achieved": achieved, "peak": peak_tflops, "unit": "TFLOP/s",
                     "frac": achieved / peak_tflops, "traffic": traffic, "traffic_basis": traffic_basis,
                     "kernel": "mp_fold_kernel (K3 Eq. 2 fold, VIADDMNMX.S16x2), config-5 graph",
                     "launches": len(folds) // len(runs),
                     "peak_basis": f"148 SM x 128 FP32 lanes x 2 ops x {f_mhz:.0f} MHz (measured SM clock under load)"},
        "minplus": {"configs": C, "layers": g.n_layers, "cell_updates": cells,
                    "cell_updates_per_s": cells / (wave_ms * 1e-3), "fold_kernel_ms": wave_ms,
                    "profiled_plan_ms": total_ms, "ms_by_kernel": by_kind,
                    "plan_ms": plan_ms, "global_cell_updates": global_cells,
                    "plan_cell_updates_per_s": global_cells / (plan_ms * 1e-3), "ranks": world,
                    "sharding": "row blocks of c_u across ranks" if world > 1 else "none",
                    "cost": r.cost, "precision": r.precision, "clocks": c,
                    "workload": f"plan_with_tables(series_parallel(seed 1, 1000 layers, bp 0.3), C={C})"},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="inception_chain@16")
    ap.add_argument("--minplus-c", type=int, default=1024)
    ap.add_argument("--minplus-runs", type=int, default=2)
    ap.add_argument("--cpu-runs", type=int, default=8)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
