#!/bin/bash
mkdir -p gpurun_out
python tools/z512_check.py new > gpurun_out/zc2.log 2>&1
AB_LIB=$PWD/libsdns_zold.so python tools/z512_check.py old >> gpurun_out/zc2.log 2>&1
python tools/z512_check.py newp 512 pencil >> gpurun_out/zc2.log 2>&1
AB_LIB=$PWD/libsdns_zold.so python tools/z512_check.py oldp 512 pencil >> gpurun_out/zc2.log 2>&1
python - >> gpurun_out/zc2.log 2>&1 <<'PY'
import numpy as np
for a, b in (("new", "old"), ("newp", "oldp")):
    x = np.load(f"gpurun_out/rhs_{a}.npy"); y = np.load(f"gpurun_out/rhs_{b}.npy")
    print(a, b, "bitwise", np.array_equal(x, y), "max", np.abs(x - y).max())
PY
rm -f gpurun_out/rhs_*.npy
bash tools/ab_libs.sh zold > gpurun_out/ab_zmir.log 2>&1
