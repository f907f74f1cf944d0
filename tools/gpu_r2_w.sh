#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/t_w.log 2>&1; echo "rc=$?" >> gpurun_out/t_w.log
python tools/small_n_probe.py > gpurun_out/small_n3.log 2>&1
