#!/bin/bash
mkdir -p gpurun_out
for v in default presplit zs64 zs128; do
  if [ $v = default ]; then unset AB_LIB; else export AB_LIB=$PWD/libsdns_$v.so; fi
  echo "== $v" >> gpurun_out/small_ab.log
  python tools/small_n_probe.py >> gpurun_out/small_ab.log 2>&1
done
