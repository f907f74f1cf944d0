#!/bin/bash
mkdir -p gpurun_out
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/launches_384.csv python tools/small_n_launches.py 384 > gpurun_out/ncu384.log 2>&1
