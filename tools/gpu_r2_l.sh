#!/bin/bash
mkdir -p gpurun_out
/usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:"k_z_fused|k_pipe_yinv|k_pipe_xinv|k_pipe_plain|k_rk_update" -c 8 -o gpurun_out/small64 -f python tools/small_n_launches.py 64 > gpurun_out/ncu_small64.log 2>&1
