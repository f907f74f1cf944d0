#!/bin/bash
# Builds an A/B variant of the product library with extra -D flags:
#   tools/build_variant.sh NAME -DSDNS_X=1 ...  ->  libsdns_NAME.so (repo root)
# Benchmark it with python bench.py --lib $PWD/libsdns_NAME.so ... (tools/ab_libs.sh)
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_1607_00850_b200/csrc"
b=build_$name; mkdir -p $b
A="-gencode arch=compute_100a,code=sm_100a"
F="$A -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $*"
K="kernels kernels_col kernels_gen context"
for f in $K; do nvcc $F -c $f.cu -o $b/$f.o & done
wait
nvcc $A -shared -cudart static -o ../../libsdns_$name.so $(for f in $K; do echo $b/$f.o; done) \
  build/comm.o build/layout.o build/iso_init.o build/runner.o build/acceptance.o -ldl -lpthread
rm -rf $b
