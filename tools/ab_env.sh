#!/bin/bash
# A/B timing over runtime switches (run from the repo root on the GPU box):
#   bash tools/ab_env.sh SDNS_XLAYOUT=0 SDNS_NO_TMA=1 ...
show() { python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['ms_per_step'], {k: round(v['avg_ms'],3) for k,v in d['passes'].items()})"; }
for v in default "$@"; do
  for rep in 1 2; do
    if [ $v = default ]; then timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline 2>/dev/null | show $v;
    else env $v timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline 2>/dev/null | show $v; fi
  done
done
