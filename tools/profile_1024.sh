#!/bin/bash
# ncu --set full capture of the n = 1024 one-GPU step's passes (one launch
# each; ncu saves and restores ~70 GB per replay pass: ~12 minutes). Summary:
# profiles/r2_ncu_full_1024.md.
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 1500 $NCU --set full --clock-control none --import-source on -k regex:"k_pipe|k_z_fused" -c 6 -o gpurun_out/full1024 -f \
  python bench.py --size 1024 --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline --no-other-configs > gpurun_out/ncu_full1024.log 2>&1; echo "ncu full rc=$?"
