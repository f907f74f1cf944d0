#!/bin/bash
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4_fft1024_launches.csv python tools/fft_api_time.py 1024 > gpurun_out/s4_fft1024_ncu.log 2>&1
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4_fft512_launches.csv python tools/fft_api_time.py 512 > gpurun_out/s4_fft512_ncu.log 2>&1
bash tools/profile_round.sh
