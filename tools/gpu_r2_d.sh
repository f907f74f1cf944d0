#!/bin/bash
# ncu full captures of the new (k_z512w) and old (k_z_fused<512>) z pass, one launch each
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
$NCU --set full --import-source on --clock-control none -k regex:k_z512w -c 1 -o gpurun_out/z512w -f \
  python tools/z512_check.py prof > gpurun_out/ncu_z512w.log 2>&1
SDNS_LIB=$PWD/libsdns_zold.so $NCU --set full --import-source on --clock-control none -k regex:k_z_fused -c 1 \
  -o gpurun_out/zold -f python tools/z512_check.py prof > gpurun_out/ncu_zold.log 2>&1
rm -f gpurun_out/rhs_*.npy
