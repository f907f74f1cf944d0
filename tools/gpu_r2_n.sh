#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/t_n.log 2>&1; echo "rc=$?" >> gpurun_out/t_n.log
python tools/small_n_probe.py > gpurun_out/small_n2.log 2>&1
bash tools/profile_round.sh > gpurun_out/profile_round.log 2>&1
