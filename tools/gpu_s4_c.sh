#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "1024 or p1_single" > gpurun_out/s4_t1024.log 2>&1; echo "rc=$?" >> gpurun_out/s4_t1024.log
tail -3 gpurun_out/s4_t1024.log
bash tools/ab_libs_n.sh 1024 noh2 > gpurun_out/s4_ab_h2.log 2>&1
cat gpurun_out/s4_ab_h2.log
timeout 300 python tools/fft_api_time.py 1024 > gpurun_out/s4_fft1024.log 2>&1; tail -5 gpurun_out/s4_fft1024.log
