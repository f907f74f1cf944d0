#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --size 1024 --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-other-configs > gpurun_out/b1024.json 2> gpurun_out/b1024.err
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_64.csv python tools/small_n_launches.py 64 > gpurun_out/ncu64.log 2>&1
