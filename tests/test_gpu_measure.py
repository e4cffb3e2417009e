"""Measured-cost producer: the document it writes is the
reference's measured-cost format, the drop-in CLI consumes it, and planning on
it equals planning on the same tables uploaded directly."""
import json
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1802_04924_b200", "bin", "parplan")


def test_measured_costs_feed_the_planner(gpu, tmp_path):
    import paper_1802_04924_b200 as P
    from paper_1802_04924_b200.measure import measure_node_costs

    g = P.builtin_model("lenet5", 32)
    dev = P.DeviceGraph.uniform(2)
    doc = measure_node_costs(g, dev, repeats=3, warmup=1, ctx=gpu.ctx)
    t = P.build_cost_tables(g, dev, gpu.ctx)
    catalog, _, _, sync, xfer = t.download()
    node = doc["node_costs"]
    assert list(node) == [g.layer_id(l) for l in range(g.n_layers)]
    for l in range(g.n_layers):
        vals = np.asarray(node[g.layer_id(l)])
        assert len(vals) == len(catalog[l]) and (vals >= sync[l]).all()
    kinds = g.kinds()
    assert all(np.asarray(node[g.layer_id(l)]).max() > 0 for l in range(g.n_layers) if kinds[l] in (1, 2, 3))

    # planning on the measured tables, two ways
    measured = [np.asarray(node[g.layer_id(l)]) for l in range(g.n_layers)]
    direct = P.plan_with_tables(g, P.upload_cost_tables(g, catalog, measured, xfer, ctx=gpu.ctx))
    # ... and the oracle on the same (uncertified FP64) tables: bit-exact
    import oracle as O

    for kind in ("port", "reference"):
        if not O.available(kind):
            continue
        want = O.Instance.builtin("lenet5", 32, kind).set_tables(catalog, measured, xfer).plan()
        assert list(direct.indices) == list(want.indices) and direct.cost == want.cost, kind
    path = tmp_path / "measured.json"
    path.write_text(json.dumps(doc))
    if not os.path.exists(CLI):
        pytest.skip("CLI not built")
    p = subprocess.run([CLI, "plan", "--model", "lenet5", "--devices", "2", "--cost-file", str(path), "--json"],
                       capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr
    out = json.loads(p.stdout)
    assert out["cost_seconds"] == direct.cost
