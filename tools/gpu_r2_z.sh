#!/bin/bash
mkdir -p gpurun_out
bash tools/ab_libs_n.sh 1024 prep1 > gpurun_out/ab_p1tma.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "1024" > gpurun_out/t_1024.log 2>&1; echo "rc=$?" >> gpurun_out/t_1024.log
