timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/tree.txt
timeout 400 tools/ab_libs.sh prev tree >> gpurun_out/tree.txt 2>&1
