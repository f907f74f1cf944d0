#!/bin/bash
# Round evidence on the GPU box (repo root): bench line, reference arm, ncu
# launch list of the bench's step, ncu --set full captures of the step's
# kernels (one launch each). Outputs in gpurun_out/; summarise here with
#   python tools/profile_summary.py r2 512 gpurun_out/launches.csv gpurun_out/full.ncu-rep gpurun_out/full_rk.ncu-rep
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-other-configs > gpurun_out/ncu_l.log 2>&1; echo "ncu list rc=$?"
timeout 1500 $NCU --set full --clock-control none --import-source on -k regex:"k_pipe|k_z_fused" -c 5 -o gpurun_out/full -f \
  python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-other-configs > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"k_rk_update" -c 4 -o gpurun_out/full_rk -f \
  python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-other-configs > gpurun_out/ncu_full_rk.log 2>&1; echo "ncu rk rc=$?"
