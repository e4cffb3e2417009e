"""paper_1802_04924_b200 — B200-native search core of the layer-wise
parallelization optimizer (arXiv 1802.04924, reference ``parplan``).

The product is ``libparplan_cuda.so`` (C ABI: ``include/parplan_c.h``; C++
drop-in headers: ``include/parplan/*.hpp``).  This package only binds it.
"""
from .capi import (  # noqa: F401
    ComputationGraph,
    Context,
    CostTables,
    CudaError,
    DeviceGraph,
    InputError,
    Layer,
    LimitError,
    ParplanError,
    PlanResult,
    PreparedPlan,
    VirtualRanks,
    shard_layout,
    ReducedGraph,
    brute_force_plan,
    build_cost_tables,
    builtin_model,
    default_context,
    device_count,
    enumerate_final,
    lib,
    plan,
    plan_with_tables,
    random_series_parallel_graph,
    series_parallel_graph,
    synthetic_instance,
    synthetic_cost_tables,
    synthetic_cost_tables64,
    upload_cost_tables,
)
