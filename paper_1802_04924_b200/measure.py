"""Measured-cost producer: per-layer, per-configuration
compute times measured on the B200, written in the reference's measured-cost
format ({"node_costs": {layer id: [seconds per catalog config]}}, io.hpp:283-342)
for apply_measured_costs / `parplan --cost-file`.

The paper estimates t_c(l, c) "by processing the layer under that configuration
multiple times on the device and measuring the average execution time",
forward and backward (PAPER.md: cost functions).  Here each configuration's
per-device shard runs through cuDNN / cuBLAS (torch, fp32): the output shard is
(N/n, C/c, H/h, W/w); convolutions and pools read the input window that shard
needs (halo included), fully-connected layers the full input features.  The
node cost written is t_c + t_s, with t_s the analytic parameter-sync time of
the same tables (cost.hpp:79-94) — the reference's node = compute + sync.
Layers without compute (input, flatten, concat) cost 0 + t_s.

    python -m paper_1802_04924_b200.measure --model vgg16 --devices 4 --out measured.json
    parplan plan --model vgg16 --devices 4 --cost-file measured.json
"""
from __future__ import annotations

import argparse
import json
from typing import Dict, Optional

import numpy as np

from . import capi as P

KIND_INPUT, KIND_CONV, KIND_POOL, KIND_FC, KIND_FLATTEN, KIND_CONCAT, KIND_SOFTMAX = range(7)


def _window(out_extent: int, kernel: int, stride: int, in_extent: int) -> int:
    """Input rows a contiguous block of `out_extent` output rows reads (halo included)."""
    return min(in_extent, (out_extent - 1) * stride + kernel)


def _shard_op(kind: int, prm, out_shape, in_shape, cfg):
    """(callable running fwd + bwd, cache key) of one configuration's shard, or None."""
    import torch
    import torch.nn.functional as F

    n, c, h, w = (int(x) for x in cfg)
    N, C, H, W = (int(x) for x in out_shape)
    bn, oc, oh, ow = max(1, N // n), max(1, C // c), max(1, H // h), max(1, W // w)
    dev = "cuda"
    if kind == KIND_CONV:
        _, kh, kw, sh, sw, ph, pw = (int(x) for x in prm)
        cin = int(in_shape[1])
        ih = _window(oh, kh, sh, int(in_shape[2]) + 2 * ph)
        iw = _window(ow, kw, sw, int(in_shape[3]) + 2 * pw)
        key = ("conv", bn, cin, ih, iw, oc, kh, kw, sh, sw)
        x = torch.randn(bn, cin, ih, iw, device=dev, requires_grad=True)
        wt = torch.randn(oc, cin, kh, kw, device=dev, requires_grad=True)

        def run():
            y = F.conv2d(x, wt, stride=(sh, sw))
            y.backward(torch.ones_like(y))
        return run, key
    if kind == KIND_POOL:
        kh, kw, sh, sw, ph, pw = (int(x) for x in prm[:6])
        ih = _window(oh, kh, sh, int(in_shape[2]) + 2 * ph)
        iw = _window(ow, kw, sw, int(in_shape[3]) + 2 * pw)
        key = ("pool", bn, oc, ih, iw, kh, kw, sh, sw)
        x = torch.randn(bn, oc, ih, iw, device=dev, requires_grad=True)

        def run():
            y = F.max_pool2d(x, (kh, kw), (sh, sw))
            y.backward(torch.ones_like(y))
        return run, key
    if kind == KIND_FC:
        fin = int(np.prod([int(v) for v in in_shape[1:]]))
        key = ("fc", bn, fin, oc)
        x = torch.randn(bn, fin, device=dev, requires_grad=True)
        wt = torch.randn(oc, fin, device=dev, requires_grad=True)

        def run():
            y = x @ wt.t()
            y.backward(torch.ones_like(y))
        return run, key
    if kind == KIND_SOFTMAX:
        key = ("softmax", bn, oc)
        x = torch.randn(bn, oc, device=dev, requires_grad=True)

        def run():
            y = torch.softmax(x, dim=1)
            y.backward(torch.ones_like(y))
        return run, key
    return None


def _time(run, repeats: int, warmup: int) -> float:
    import torch

    for _ in range(warmup):
        run()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    start.record()
    for _ in range(repeats):
        run()
    end.record()
    end.synchronize()
    return start.elapsed_time(end) / repeats * 1e-3  # seconds


def measure_node_costs(graph: P.ComputationGraph, devices: P.DeviceGraph, repeats: int = 10, warmup: int = 3,
                       ctx: Optional[P.Context] = None) -> Dict:
    """{"node_costs": {layer id: [t_c + t_s per catalog config]}} for `graph` on `devices`."""
    tables = P.build_cost_tables(graph, devices, ctx)
    catalog, _, _, sync, _ = tables.download()
    kinds, params, shapes = graph.kinds(), graph.params(), graph.shapes()
    src, dst, _ = graph.edges()
    first_in = {}
    for e in range(len(dst)):
        first_in.setdefault(int(dst[e]), int(src[e]))
    cache: Dict = {}
    out: Dict = {}
    for l in range(graph.n_layers):
        in_shape = shapes[first_in.get(l, l)]
        vals = []
        for i, cfg in enumerate(catalog[l]):
            op = _shard_op(int(kinds[l]), params[l], shapes[l], in_shape, cfg)
            tc = 0.0
            if op is not None:
                run, key = op
                if key not in cache:
                    cache[key] = _time(run, repeats, warmup)
                tc = cache[key]
            vals.append(tc + float(sync[l][i]))
        out[graph.layer_id(l)] = vals
    return {"node_costs": out}


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    src = ap.add_mutually_exclusive_group(required=True)
    src.add_argument("--model", help="builtin model (lenet5, alexnet, vgg16, inception_chain[(K)])")
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--devices", type=int, default=1)
    ap.add_argument("--repeats", type=int, default=10)
    ap.add_argument("--out", required=True)
    a = ap.parse_args(argv)
    g = P.builtin_model(a.model, a.batch)
    doc = measure_node_costs(g, P.DeviceGraph.uniform(a.devices), repeats=a.repeats)
    with open(a.out, "w") as f:
        json.dump(doc, f, indent=2)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
