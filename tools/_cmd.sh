timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/pk.txt
for r in 1 2; do for v in prev pk; do cp _ab/lib_$v.so paper_1802_04924_b200/libparplan_cuda.so; echo "$v $(python tools/mp_ab.py 2>&1 | tail -1)" >> gpurun_out/pk.txt; done; done
