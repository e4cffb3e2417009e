#!/bin/bash
# Round profile capture on the GPU box (one GPU; never multi-rank under ncu).
#   1. plain bench run (must exit 0 before any ncu pass)
#   2. launch list of the same bench command (per-launch gpu__time_duration)
#   3. --set full of the dominant min-plus fold kernel and of the fused plan kernel
set -e
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 > gpurun_out/bench_plain.json 2> gpurun_out/bench_plain.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 > gpurun_out/ncu_launches.log 2>&1 || true
ncu --set full --import-source on --clock-control none -k regex:mp_fold_kernel -s 40 -c 1 \
    -o gpurun_out/mp_fold_full -f python tools/profile_run.py minplus 1024 200 > gpurun_out/ncu_mp.log 2>&1 || true
ncu --set full --import-source on --clock-control none -k regex:dp_fused_kernel -s 2 -c 1 \
    -o gpurun_out/fused_full -f python tools/profile_run.py search > gpurun_out/ncu_fused.log 2>&1 || true
ls -la gpurun_out
