#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_generic_n.py -m gpu -q -x > gpurun_out/s4_tpar.log 2>&1; echo "rc=$?" >> gpurun_out/s4_tpar.log
tail -3 gpurun_out/s4_tpar.log
timeout 300 python tools/small_n_steps.py > gpurun_out/s4_small.log 2>&1; cat gpurun_out/s4_small.log
timeout 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4_small_launches.csv python tools/small_n_launches.py 64 > /dev/null 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-1024 > gpurun_out/s4_bench2.json 2> gpurun_out/s4_bench2.err; echo "bench rc=$?"
