#!/bin/bash
# Round-end evidence on the GPU box: bench line, reference arm, ncu launch list.
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-other-configs > gpurun_out/ncu_l.log 2>&1; echo "ncu rc=$?"
