#!/bin/bash
# A/B of prebuilt library variants _ab/lib_<name>.so, interleaved over two
# rounds: tools/lib_ab.sh "<command>" base new ...
set -u
cmd=$1; shift
cp paper_1802_04924_b200/libparplan_cuda.so /tmp/lib_current.so
for r in 1 2; do
  for v in "$@"; do
    cp _ab/lib_$v.so paper_1802_04924_b200/libparplan_cuda.so
    echo "== $v (round $r)"
    bash -c "$cmd" 2>&1
  done
done
cp /tmp/lib_current.so paper_1802_04924_b200/libparplan_cuda.so
