#!/bin/bash
# A/B timing of library variants on the GPU box (run from the repo root):
#   tools/build_variant.sh NAME -DFLAG=...   (here)   then
#   gpurun -- 'bash tools/ab_libs.sh NAME1 NAME2'  -> per-pass ms for default + variants
mkdir -p gpurun_out
show() { python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['ms_per_step'], {k: round(v['avg_ms'],3) for k,v in d['passes'].items()})"; }
for v in default "$@"; do
  if [ $v = default ]; then LIB=""; else LIB="--lib $PWD/libsdns_$v.so"; fi
  for rep in 1 2; do
    timeout 300 python bench.py $LIB --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-other-configs 2>/dev/null | show $v
  done
done
