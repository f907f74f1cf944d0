show() { python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['ms_per_step'], {k: round(v['avg_ms'],3) for k,v in d['passes'].items()})"; }
for v in default nofft; do
  if [ $v = default ]; then unset SDNS_LIB; else export SDNS_LIB=$PWD/libsdns_$v.so; fi
  for n in 256 512; do
    timeout 300 python bench.py --n $n --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline 2>/dev/null | show "$v-$n"
  done
done
