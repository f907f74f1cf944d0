for v in default cs4l; do
  if [ $v = default ]; then unset SDNS_LIB; else export SDNS_LIB=$PWD/libsdns_$v.so; fi
  timeout 900 python bench.py --n 1024 --steps 2 --warmup 2 --e2e-steps 1 --no-cpu-baseline 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], {k: round(v['avg_ms'],2) for k,v in d['passes'].items()})"
done
