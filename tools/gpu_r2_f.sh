#!/bin/bash
mkdir -p gpurun_out
python tools/small_n_probe.py > gpurun_out/small_n.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/t_all.log 2>&1; echo "rc=$?" >> gpurun_out/t_all.log
