#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/t_q.log 2>&1; echo "rc=$?" >> gpurun_out/t_q.log
timeout 1200 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:"k_pipe_xinv|k_z_fused|k_pipe_yinv" -c 3 -o gpurun_out/full1024 -f \
  python bench.py --size 1024 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-other-configs > gpurun_out/ncu1024.log 2>&1
