timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/enr.txt
timeout 400 tools/ab_libs.sh prev enr >> gpurun_out/enr.txt 2>&1
