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
os.environ.setdefault("NCCL_DEBUG", "WARN")

# stdout carries exactly one JSON line: libraries that print to fd 1 (NCCL's
# version banner, ...) go to stderr; the line is written to the saved stdout
_JSON_OUT = os.fdopen(os.dup(1), "w")
os.dup2(2, 1)


def emit(line: dict) -> None:
    _JSON_OUT.write(json.dumps(line) + "\n")
    _JSON_OUT.flush()

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
        "config": config_of(model, batch, D),
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
    emit(line)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

GOLDEN = os.path.join(ROOT, "tests", "golden")
# real-model workloads reported beside the headline (BASELINE configs 1-4 + the
# 13-module chain, the nearest to Inception-v3's 120 nodes)
MODELS = [("inception_chain", 16), ("inception_chain", 64), ("inception_chain(13)", 16), ("vgg16", 16),
          ("alexnet", 4), ("lenet5", 4)]


def golden_builtin(model, D):
    with open(os.path.join(GOLDEN, "reference_golden.json")) as f:
        for c in json.load(f)["builtins"]:
            if c["model"] == model and c["devices"] == D:
                return c
    return None


def config_of(model, batch, D):
    """The config dict both arms print (identical keys and values)."""
    wl = f"plan(inception_chain(12)@{D})" if model == "inception_chain" else f"plan({model}@{D})"
    return {"workload": wl, "model": model, "batch": batch, "devices": D}


def time_prepared(P, prep, stream, flush, steps, warmup):
    import torch

    for _ in range(warmup):
        flush.zero_()
        prep.launch()
        prep.fetch()
    ms = []
    for _ in range(steps):
        flush.zero_()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        prep.launch()
        s1.record(stream)
        r = prep.fetch()
        ms.append(s0.elapsed_time(s1))
    return ms, r


def model_sweep(P, ctx, stream, flush, args):
    """Device ms (prepared plan, inputs resident) and e2e ms (pp_plan with host
    buffers) per real-model workload, each checked against the reference golden
    (indices + cost as hex-float; tests/golden/make_golden.py)."""
    import torch

    out = {}
    for model, D in MODELS:
        g = P.builtin_model(model, 32)
        dev = P.DeviceGraph.uniform(D)
        prep = P.PreparedPlan(g, devices=dev, ctx=ctx)
        dms, r = time_prepared(P, prep, stream, flush, args.steps, args.warmup)
        e2e = []
        for k in range(args.warmup + args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = P.plan(g, dev, ctx=ctx)
            if k >= args.warmup:
                e2e.append((time.perf_counter() - t0) * 1e3)
        gold = golden_builtin(model, D)
        ok = gold is not None and [int(x) for x in r.indices] == gold["indices"] and float(r.cost).hex() == gold["cost"] \
            and [int(x) for x in res.indices] == gold["indices"] and float(res.cost).hex() == gold["cost"]
        out[f"{model}@{D}"] = {
            "layers": g.n_layers, "edges": g.n_edges, "device_ms": statistics.mean(dms),
            "device_ms_median": statistics.median(dms), "e2e_ms": statistics.mean(e2e),
            "e2e_ms_median": statistics.median(e2e), "cost": r.cost, "waves": r.waves,
            "matches_reference": bool(ok),
            "reference_cpu_s": gold.get("reference_cpu_s") if gold else None}
        del prep
    return out


def dropin_latency(args):
    """bin/plan_bench: parplan::plan(graph, DeviceGraph::uniform(D)) through the
    drop-in C++ API with a fresh graph per call (acceptance C5's measurement)."""
    exe = os.path.join(ROOT, "paper_1802_04924_b200", "bin", "plan_bench")
    if not os.path.exists(exe):
        return {"unavailable": "paper_1802_04924_b200/bin/plan_bench not built"}
    try:
        cp = subprocess.run([exe, str(max(args.steps, 10)), "3"], capture_output=True, text=True, timeout=600,
                            env=dict(os.environ, PARPLAN_DEVICE=os.environ.get("LOCAL_RANK", "0")))
        rows = [json.loads(x) for x in cp.stdout.splitlines() if x.startswith("{")]
    except Exception as exc:
        return {"unavailable": f"plan_bench failed: {exc}"}
    out = {}
    for r in rows:
        out[f"{r['kind']}:{r['workload']}"] = {"median_ms": r["median_ms"], "mean_ms": r["mean_ms"], "cost": r["cost"]}
    return out


def table_build(P, ctx):
    """K1/K2 standalone (pp_tables_build) at I64: partition pairs per second
    (one (p, q) pair of the reference's transfer_profile walk,
    cost.hpp:103-131 — Σ over xfer cells of total(c_src) * total(c_dst)) and
    GB/s of the table bytes written (8 B per xfer cell, 24 B per node cell)."""
    import numpy as np

    g = P.builtin_model("inception_chain", 32)
    dev = P.DeviceGraph.uniform(64)
    ms = []
    t = None
    for _ in range(6):
        t = P.build_cost_tables(g, dev, ctx)
        ms.append(t.build_ms)
    cat = t.download()[0]
    tot = [np.prod(np.asarray(c, np.int64).reshape(-1, 4), axis=1) for c in cat]
    es, ed, _ = g.edges()
    pairs = sum(float(tot[s].sum()) * float(tot[d].sum()) for s, d in zip(es, ed))
    xcells = sum(len(tot[s]) * len(tot[d]) for s, d in zip(es, ed))
    ncells = sum(len(x) for x in tot)
    best = min(ms[1:])
    bytes_ = 8.0 * xcells + 24.0 * ncells
    return {"workload": "build_cost_tables(inception_chain(12)@64)", "kernel": "build_tables_kernel (K1 + K2)",
            "ms": best, "ms_all": ms[1:], "partition_pairs": pairs, "pairs_per_s": pairs / (best * 1e-3),
            "xfer_cells": xcells, "bytes_written": bytes_, "achieved_gbs": bytes_ / (best * 1e-3) / 1e9,
            "hbm_peak_gbs": peaks().get("hbm_gbs"),
            "note": "integer-issue bound (SURVEY §8(d)); GB/s reported as §8(d) asks, judged by pairs/s"}


def committed_traffic(kernel):
    """DRAM bytes (read + write) of one launch of `kernel` from the newest
    committed ncu --set full summary under profiles/ (the roofline's traffic)."""
    import csv
    import glob

    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_full_summary.csv")), reverse=True):
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


def minplus_point(P, ctx, stream, C, runs, check):
    """Config-5 synthetic graph (1000 layers, bp 0.3, seed 1), C configs per
    layer, exact int32 fixed point.  C <= 1024: the reference's draw order
    (host mt19937_64, oracle.hpp:121-185), checked against the REAL reference's
    result (tests/golden/reference_synth_C{C}.json); larger C: the device
    generator, checked against the generic int32 fold on the same tables."""
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    gold_path = os.path.join(GOLDEN, f"reference_synth_C{C}.json")
    if C <= 1024 and os.path.exists(gold_path):
        g, t = P.synthetic_instance(1, 1000, C, 0.3, ctx=ctx)
        tables = "reference draw order (host mt19937_64, oracle.hpp:121-185)"
    else:
        g = P.series_parallel_graph(1, 1000, 0.3)
        t = P.synthetic_cost_tables(g, C, seed=1, ctx=ctx)
        tables = "device generator (splitmix64, values k/64, k in [0, 640])"
    prep = P.PreparedPlan(g, tables=t, ctx=ctx)
    prep.launch()
    r = prep.fetch()
    sched = g.schedule()[0]
    folds = [rec for rec in sched if rec[0] == 0]
    global_cells = float(C) ** 3 * len(folds)
    merge_cells = float(C) ** 2 * (len(sched) - len(folds))
    runs_ = [prep.profile() for _ in range(runs)]
    plan_ms = []
    for _ in range(3):
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s0.record(stream)
        prep.launch()
        s1.record(stream)
        prep.fetch()
        plan_ms.append(s0.elapsed_time(s1))
    plan_ms = min(plan_ms)
    if world > 1:
        from paper_1802_04924_b200 import distributed as PD

        plan_ms = PD.max_over_ranks(plan_ms, device="cuda")
    by_kind = {}
    for run in runs_:
        for kind, ms, _ in run:
            by_kind[kind] = by_kind.get(kind, 0.0) + ms / len(runs_)
    fold = [(ms, w) for run in runs_ for kind, ms, w in run if kind in ("mp_fold", "mp_chain")]
    fold_ms = sum(ms for ms, _ in fold) / len(runs_)
    cells = sum(w for _, w in fold) / len(runs_)
    merge = [(ms, w) for run in runs_ for kind, ms, w in run if kind == "mp_merge"]
    merge_ms = sum(ms for ms, _ in merge) / len(runs_)
    mcells = sum(w for _, w in merge) / len(runs_)
    del prep
    out = {"configs": C, "layers": g.n_layers, "tables": tables, "fold_kernel_ms": fold_ms,
           "fold_launches": len(fold) // len(runs_), "cell_updates": cells, "plan_ms": plan_ms,
           "global_cell_updates": global_cells, "ms_by_kernel": by_kind, "cost": r.cost, "precision": r.precision,
           "k4_merge": {"kernel": "mp_merge_kernel (Eq. 3, int32 add + column minima)", "ms": merge_ms,
                        "cells": mcells, "bytes": 12.0 * mcells,
                        "achieved_gbs": 12.0 * mcells / (merge_ms * 1e-3) / 1e9 if merge_ms else None,
                        "hbm_peak_gbs": peaks().get("hbm_gbs")} if mcells else None}
    if check and os.path.exists(gold_path) and "reference draw order" in tables:
        with open(gold_path) as f:
            gold = json.load(f)
        out["matches_reference"] = bool([int(x) for x in r.indices] == gold["indices"] and float(r.cost).hex() == gold["cost"])
        out["reference_cpu_s"] = gold["reference_cpu_s"]
    elif check:
        ctx.set_kernel_policy("generic")  # the same device tables through the generic tiled int32 fold
        try:
            b = P.plan_with_tables(g, t)
            out["matches_generic"] = bool(list(b.indices) == list(r.indices) and b.cost == r.cost)
            out["generic_ms"] = b.device_ms
        finally:
            ctx.set_kernel_policy("auto")
    del t
    return out


def minplus_fp64(P, ctx, stream, C, check):
    """The FP64 large-table fold (minplus64.cuh) on the config-5 graph with
    non-dyadic FP64 tables (what measured costs look like; the fixed-point
    certificate rejects them): cells/s against the FP64-pipe roofline
    (64 DADD lane-ops/clk/SM measured, profiles/r02_microbench_fp64_tput.log;
    2 FP64-pipe ops per cell: DADD + DSETP)."""
    import torch

    g = P.series_parallel_graph(1, 1000, 0.3)
    t = P.synthetic_cost_tables64(g, C, seed=1, ctx=ctx)
    prep = P.PreparedPlan(g, tables=t, ctx=ctx)
    prep.launch()
    r = prep.fetch()
    prof = prep.profile()
    fold_ms = sum(ms for k, ms, _ in prof if k == "mp64_fold")
    cells = sum(w for k, _, w in prof if k == "mp64_fold")
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s0.record(stream)
    prep.launch()
    s1.record(stream)
    prep.fetch()
    plan_ms = s0.elapsed_time(s1)
    del prep
    peak = 148 * 32 * 1965e6
    out = {"configs": C, "tables": "device generator, FP64 (k + u)/64, 53-bit u (uncertified)", "precision": r.precision,
           "fold_kernel_ms": fold_ms, "cell_updates": cells, "cell_updates_per_s": cells / (fold_ms * 1e-3) if fold_ms else None,
           "fp64_cell_peak_per_s": peak, "fold_frac": cells / (fold_ms * 1e-3) / peak if fold_ms else None,
           "peak_basis": "148 SM x 64 FP64 lane-ops/clk (measured) / 2 ops per cell x 1965 MHz",
           "plan_ms": plan_ms, "cost": r.cost}
    if check:
        ctx.set_kernel_policy("generic")
        try:
            b = P.plan_with_tables(g, t)
            out["matches_generic"] = bool(list(b.indices) == list(r.indices) and b.cost == r.cost)
            out["generic_ms"] = b.device_ms
        finally:
            ctx.set_kernel_policy("auto")
    del t
    return out


def minplus(P, ctx, args, stream, sm_mhz):
    """Min-plus sweep; the headline roofline is the C=1024 point's mp_fold_kernel."""
    points = {}
    import torch

    def mem():
        free, total = torch.cuda.mem_get_info()
        return f"device memory free {free / 2**30:.1f} of {total / 2**30:.1f} GiB"

    for C in args.minplus_sweep:
        ctx.release_pools()  # the previous point's one-shot (generic check) plan pool
        torch.cuda.empty_cache()
        try:
            points[str(C)] = minplus_point(P, ctx, stream, C, args.minplus_runs, check=not args.no_check)
        except Exception as exc:  # report, keep the line
            points[str(C)] = {"error": str(exc)[:300] + "; " + mem()}
    f_mhz = sm_mhz or peaks().get("sm_max_mhz", 1965.0)
    peak_tflops = 148 * 128 * 2 * f_mhz * 1e6 / 1e12  # FP32 CUDA-core: 2 ops (add + min) per cell update per lane-clock
    for pt in points.values():
        if "fold_kernel_ms" in pt and pt["fold_kernel_ms"] and pt.get("precision") != "fp64":
            pt["fold_frac"] = 2.0 * pt["cell_updates"] / (pt["fold_kernel_ms"] * 1e-3) / 1e12 / peak_tflops
            pt["plan_frac"] = 2.0 * pt["global_cell_updates"] / (pt["plan_ms"] * 1e-3) / 1e12 / peak_tflops
            pt["plan_cell_updates_per_s"] = pt["global_cell_updates"] / (pt["plan_ms"] * 1e-3)
    if args.fp64_c:
        ctx.release_pools()
        torch.cuda.empty_cache()
        try:
            points[f"fp64_{args.fp64_c}"] = minplus_fp64(P, ctx, stream, args.fp64_c, check=not args.no_check)
        except Exception as exc:
            points[f"fp64_{args.fp64_c}"] = {"error": str(exc)[:300] + "; " + mem()}
    head = points.get(str(args.minplus_c)) or next(iter(points.values()), {})
    traffic, basis = committed_traffic("mp_fold_kernel")
    roof = None
    if head.get("fold_kernel_ms"):
        achieved = 2.0 * head["cell_updates"] / (head["fold_kernel_ms"] * 1e-3) / 1e12
        launches = max(1, head["fold_launches"])
        roof = {"bound": "fp32", "achieved": achieved, "peak": peak_tflops, "unit": "TFLOP/s",
                "frac": achieved / peak_tflops, "traffic": traffic, "traffic_basis": basis,
                "kernel": f"mp_fold_kernel (K3 Eq. 2 fold, VIADDMNMX.U16x2), config-5 graph at C={head['configs']}",
                "launches": launches, "algorithmic": "2 ops (add + min) per cell update; cells = sum nu*nw*nv",
                "peak_basis": f"148 SM x 128 FP32 lanes x 2 ops x {f_mhz:.0f} MHz (SM clock sampled under load)",
                "plan_frac": head.get("plan_frac")}
    return roof, points


def sharded(P, args, local, stream, flush):
    """One plan row-sharded across all ranks (pp_context_attach_comm: rows of
    c_u in blocks, NCCL all-gathers of derived t2 at re-association points and
    of the final edges, the unwind reading argmin rows from their owner rank
    through CUDA IPC).  Device ms = max over ranks (strong scaling: the total
    work is fixed as N grows)."""
    import torch

    from paper_1802_04924_b200 import distributed as PD

    world = int(os.environ.get("WORLD_SIZE", "1"))
    torch.cuda.empty_cache()
    sctx = P.Context(local, stream=stream.cuda_stream)
    PD.attach(sctx)
    out = {"ranks": world}
    # Inception-v3 stand-in on 64 virtual devices (BASELINE config 4)
    g = P.builtin_model("inception_chain", 32)
    prep = P.PreparedPlan(g, devices=P.DeviceGraph.uniform(64), ctx=sctx)
    ms, r = time_prepared(P, prep, stream, flush, args.steps, args.warmup)
    gold = golden_builtin("inception_chain", 64)
    out["inception_chain@64"] = {
        "device_ms": PD.max_over_ranks(statistics.mean(ms), device="cuda"),
        "matches_reference": bool(gold and [int(x) for x in r.indices] == gold["indices"]
                                  and float(r.cost).hex() == gold["cost"]),
        "note": "K1 edge-sharded + broadcast, K2 on every rank, row-sharded DP, distributed unwind; latency-bound, sharding is not expected to help (SURVEY §8e)"}
    del prep
    # the min-plus config-5 graph at C = shard_c
    C = args.shard_c
    g = P.series_parallel_graph(1, 1000, 0.3)
    t = P.synthetic_cost_tables(g, C, seed=1, ctx=sctx)
    prep = P.PreparedPlan(g, tables=t, ctx=sctx)
    prep.launch()
    r = prep.fetch()
    best = 1e30
    for _ in range(2):
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        prep.launch()
        s1.record(stream)
        prep.fetch()
        best = min(best, s0.elapsed_time(s1))
    plan_ms = PD.max_over_ranks(best, device="cuda")
    folds = sum(1 for rec in g.schedule()[0] if rec[0] == 0)
    cells = float(C) ** 3 * folds
    prof = prep.profile()
    ag = sum(ms for k, ms, _ in prof if k == "allgather")
    agb = sum(w for k, _, w in prof if k == "allgather")
    peak = 148 * 128 * 2 * 1965e6 * world / 1e12
    out[f"minplus_C{C}"] = {"plan_ms": plan_ms, "cell_updates": cells, "cell_updates_per_s": cells / (plan_ms * 1e-3),
                            "plan_frac_of_n_gpus": 2.0 * cells / (plan_ms * 1e-3) / 1e12 / peak,
                            "allgather_ms_profiled": ag, "allgather_bytes": agb, "cost": r.cost,
                            "sharding": "row blocks of c_u; derived t2 all-gathered before its fold"}
    del prep, t
    return out


def run_ours(args):
    import numpy as np  # noqa: F401
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
    g = P.builtin_model(model, batch)
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
    # whole-job: N ranks each search their own replica in the max-rank time
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
    # the same call with the plan cache off: every call prepares from scratch
    # (catalogs and schedule still cached per graph)
    os.environ["PARPLAN_PLAN_CACHE"] = "0"
    e2e_nc = []
    for k in range(args.warmup + args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = P.plan(g, dev, ctx=ctx)
        if k >= args.warmup:
            e2e_nc.append((time.perf_counter() - t0) * 1e3)
    del os.environ["PARPLAN_PLAN_CACHE"]
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
    pw, _ = time_prepared(P, P.PreparedPlan(g, tables=t_built, ctx=ctx), stream, flush, args.steps, args.warmup)
    gold = golden_builtin(model if model != "inception_chain" else "inception_chain", D)

    line = {
        "metric": METRIC, "value": value, "unit": "ms", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": max(dev_ms) if world == 1 else value * world, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": value / PAPER_MS, "dtype": "f64",
        "data": "synthetic (builtin model graph, analytic cost tables; each rank searches its own replica)",
        "config": config_of(model, batch, D),
        "config_detail": {"layers": g.n_layers, "edges": g.n_edges, "l2": "256 MiB write between timed steps",
                          "parallelism": f"replicas x{world}" if world > 1 else "single GPU"},
        "e2e": {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "call": "pp_plan(ctx, graph, device_desc, k_bound, host indices), repeated: the library's plan "
                        "cache replays a prepared plan -- H2D of the descriptor image (graph + device inputs), "
                        "table build, search, D2H of the result every call (see dropin_e2e for parplan::plan() "
                        "with a fresh graph per call)",
                "no_plan_cache_ms": statistics.mean(e2e_nc)},
        "gpu_launches": launches,
        "plan_with_tables_ms": statistics.mean(pw),
        "result": {"cost": r.cost, "node_eliminations": r.node_eliminations, "edge_eliminations": r.edge_eliminations,
                   "waves": r.waves, "precision": r.precision,
                   "matches_reference": bool(gold and [int(x) for x in r.indices] == gold["indices"]
                                             and float(r.cost).hex() == gold["cost"])},
        "search_kernels": kern,
        "clocks": clk.summary(),
    }
    if not args.quick:
        line["models"] = model_sweep(P, ctx, stream, flush, args)
        if rank == 0:
            line["dropin_e2e"] = dropin_latency(args)
        line["k1_table_build"] = table_build(P, ctx)

    # ---- min-plus roofline and sweep (config-5 synthetic graph) ----------------------------
    if args.minplus_sweep:
        with Clocks(local) as mclk:
            roof, points = minplus(P, ctx, args, stream, None)
        mc = mclk.summary()
        if mc.get("sm_mhz"):  # re-base the peak on the clock sampled under the min-plus load
            f = mc["sm_mhz"]
            pk = 148 * 128 * 2 * f * 1e6 / 1e12
            for pt in points.values():
                if pt.get("fold_kernel_ms") and pt.get("precision") != "fp64":
                    pt["fold_frac"] = 2.0 * pt["cell_updates"] / (pt["fold_kernel_ms"] * 1e-3) / 1e12 / pk
                    pt["plan_frac"] = 2.0 * pt["global_cell_updates"] / (pt["plan_ms"] * 1e-3) / 1e12 / pk
            if roof:
                roof["peak"] = pk
                roof["frac"] = roof["achieved"] / pk
                roof["plan_frac"] = points.get(str(args.minplus_c), {}).get("plan_frac")
                roof["peak_basis"] = f"148 SM x 128 FP32 lanes x 2 ops x {f:.0f} MHz (SM clock sampled under the min-plus load)"
        if roof:
            line["roofline"] = roof
        line["minplus"] = {"points": points, "clocks": mc,
                           "workload": "plan_with_tables(series_parallel(seed 1, 1000 layers, bp 0.3), C configs)"}

    # ---- N > 1: the row-sharded plans (one plan across all ranks, NCCL) -----------------
    if world > 1 and not args.no_shard:
        try:
            line["sharded"] = sharded(P, args, local, stream, flush)
        except Exception as exc:  # report, keep the line
            line["sharded"] = {"error": str(exc)[:300]}

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
        small = {}
        for m, d in (("lenet5", 4), ("alexnet", 4)):  # per-call latency where fixed overheads dominate
            _, ts, _ = reference_plan_ms(m, 32, d, 20, 3)
            small[f"{m}@{d}"] = statistics.median(ts)
        line["cpu_baseline"]["small_models_ms"] = small
        line["result"]["matches_cpu_reference"] = bool(
            list(res_ref.indices) == list(r.indices) and res_ref.cost == r.cost)
    if rank == 0:
        emit(line)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="inception_chain@16")
    ap.add_argument("--minplus-c", type=int, default=1024, help="the sweep point the headline roofline is quoted on")
    ap.add_argument("--minplus-sweep", type=lambda x: [int(c) for c in x.split(",") if c], default=[1024, 2048, 4096])
    ap.add_argument("--minplus-runs", type=int, default=2)
    ap.add_argument("--no-check", action="store_true", help="skip the min-plus parity checks")
    ap.add_argument("--fp64-c", type=int, default=1024, help="configs of the FP64 large-fold point (0: skip)")
    ap.add_argument("--quick", action="store_true", help="headline only (no model sweep / drop-in / K1)")
    ap.add_argument("--shard-c", type=int, default=4096, help="N > 1: configs of the row-sharded min-plus plan")
    ap.add_argument("--no-shard", action="store_true", help="N > 1: skip the row-sharded plans")
    ap.add_argument("--cpu-runs", type=int, default=8)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
