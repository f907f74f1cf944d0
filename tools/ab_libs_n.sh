#!/bin/bash
# ab_libs.sh at another grid size: bash tools/ab_libs_n.sh SIZE NAME...
mkdir -p gpurun_out
size=$1; shift
show() { python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['ms_per_step'], {k: round(v['avg_ms'],3) for k,v in d['passes'].items()})"; }
for v in default "$@"; do
  if [ $v = default ]; then LIB=""; else LIB="--lib $PWD/libsdns_$v.so"; fi
  timeout 600 python bench.py $LIB --size $size --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-other-configs 2>/dev/null | show $v
done
