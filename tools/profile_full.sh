#!/bin/bash
# One ncu --set full capture of the step's kernels (one launch each: stage 0
# of a warm step), for profiles/<round>_ncu_full_512.md. Run on the GPU box
# after tools/profile_round.sh exited 0.
mkdir -p gpurun_out
timeout 300 python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/plain_full.log 2>&1; echo "plain rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_pipe|k_z_fused" -c 5 -o gpurun_out/full_r1 -f python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-other-configs > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rk_update" -c 4 -o gpurun_out/full_r1_rk -f python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-other-configs > gpurun_out/ncu_full_rk.log 2>&1; echo "ncu rk rc=$?"
