#!/bin/bash
# z512w A/B: correctness vs the two-warp kernel, per-pass timing, parity at 512^3
mkdir -p gpurun_out
python tools/z512_check.py new > gpurun_out/zc.log 2>&1
SDNS_LIB=$PWD/libsdns_zold.so python tools/z512_check.py old >> gpurun_out/zc.log 2>&1
python tools/z512_check.py newp 512 pencil >> gpurun_out/zc.log 2>&1
SDNS_LIB=$PWD/libsdns_zold.so python tools/z512_check.py oldp 512 pencil >> gpurun_out/zc.log 2>&1
python - >> gpurun_out/zc.log 2>&1 <<'PY'
import numpy as np
for a, b in (("new", "old"), ("newp", "oldp"), ("new", "newp")):
    x = np.load(f"gpurun_out/rhs_{a}.npy"); y = np.load(f"gpurun_out/rhs_{b}.npy")
    print(a, b, "rel diff", np.linalg.norm(x - y) / np.linalg.norm(y), "max", np.abs(x - y).max())
PY
rm -f gpurun_out/rhs_*.npy
bash tools/ab_libs.sh zold > gpurun_out/ab_z.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -k "config3_512 or 512_pipeline_variants" > gpurun_out/t3.log 2>&1; echo "t3 rc=$?" >> gpurun_out/t3.log
