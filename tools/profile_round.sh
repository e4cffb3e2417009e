#!/bin/bash
# Round profile capture on the GPU box (one GPU; never multi-rank under ncu).
#   1. plain bench run (must exit 0 before any ncu pass)
#   2. launch lists: the headline search (bench --quick) and the C=1024
#      min-plus bench leg (per-launch gpu__time_duration, serialised)
#   3. --set full of the min-plus kernels (mp_fold on a wide and a narrow
#      launch, mp_chain, mp_prep, mp_merge, mp_minima, the FP64 mp64_fold), the
#      K1/K2 table build at I64 and the fused plan kernel (I16)
set -e
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_plain.json 2> gpurun_out/bench_plain.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv \
    python bench.py --quick --no-cpu --minplus-sweep "" --steps 3 --warmup 3 > gpurun_out/ncu_launches.log 2>&1 || true
ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/launches_mp1024.csv \
    python bench.py --quick --no-cpu --no-check --minplus-sweep 1024 --minplus-runs 1 --steps 3 --warmup 3 \
    > gpurun_out/ncu_launches_mp.log 2>&1 || true
full() { # name kernel-regex skip -- command
  local name=$1 k=$2 s=$3; shift 4
  ncu --set full --import-source on --clock-control none -k "regex:$k" -s "$s" -c 1 -o "gpurun_out/$name" -f "$@" \
      > "gpurun_out/ncu_$name.log" 2>&1 || true
}
full mp_fold_wide_full mp_fold_kernel 0 -- python tools/mp_once.py 1024
full mp_fold_full mp_fold_kernel 10 -- python tools/mp_once.py 1024
full mp_chain_full mp_chain_kernel 0 -- python tools/mp_once.py 1024
full mp64_fold_full mp64_fold_kernel 0 -- python tools/fp64_check.py 1024 120
full mp_prep_full mp_prep_kernel 0 -- python tools/mp_once.py 1024
full mp_merge_full mp_merge_kernel 0 -- python tools/mp_once.py 1024
full mp_minima_full mp_minima_kernel 0 -- python tools/mp_once.py 1024
full k1_build_i64_full build_tables_kernel 1 -- python tools/build_tables_once.py inception_chain@64
full fused_full dp_fused_kernel 2 -- python tools/profile_run.py search
ls -la gpurun_out
