#!/bin/bash
mkdir -p gpurun_out
( time timeout 900 python bench.py --steps 20 --warmup 5 ) > gpurun_out/bench_g.json 2> gpurun_out/bench_g.err; echo "bench rc=$?" >> gpurun_out/bench_g.err
timeout 1500 python -m pytest tests -m gpu -q -x -k "transpose_modes or pipeline_variants or generic_length_decompositions or multiprocess or runner or checkpoint" > gpurun_out/t_g.log 2>&1; echo "rc=$?" >> gpurun_out/t_g.log
