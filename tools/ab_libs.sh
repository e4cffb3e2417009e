#!/bin/bash
# A/B of prebuilt library variants in _ab/lib_<name>.so (interleaved rounds):
# per variant, the fused-kernel phase medians of tools/ab_fused.py and the
# build-phase barrier trace.   tools/ab_libs.sh base noinl
set -u
cp paper_1802_04924_b200/libparplan_cuda.so /tmp/lib_current.so
for r in 1 2; do
  for v in "$@"; do
    cp _ab/lib_$v.so paper_1802_04924_b200/libparplan_cuda.so
    echo "== $v (round $r)"
    python tools/ab_fused.py '{"PARPLAN_GRID_BARRIER": ["1"]}' 2>&1 | tail -1
    python tools/wave_trace.py inception_chain@16 2>&1 | grep "^build:" | tail -1
  done
done
cp /tmp/lib_current.so paper_1802_04924_b200/libparplan_cuda.so
