for v in default zt64 zt128; do
  if [ $v = default ]; then unset SDNS_LIB; else export SDNS_LIB=$PWD/libsdns_$v.so; fi
  for n in 64 128 256; do
    timeout 300 python bench.py --n $n --steps 20 --warmup 5 --e2e-steps 1 --no-cpu-baseline 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', $n, round(d['ms_per_step'],3), {k: round(v['avg_ms']*1000,1) for k,v in d['passes'].items() if k=='z_fused'})"
  done
done
