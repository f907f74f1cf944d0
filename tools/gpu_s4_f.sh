#!/bin/bash
mkdir -p gpurun_out
bash tools/ab_libs_n.sh 1024 noflat > gpurun_out/s4_ab_flat1024.log 2>&1; cat gpurun_out/s4_ab_flat1024.log
bash tools/ab_libs_n.sh 512 noflat > gpurun_out/s4_ab_flat512.log 2>&1; cat gpurun_out/s4_ab_flat512.log
bash tools/ab_libs_n.sh 512 noflat > gpurun_out/s4_ab_flat512b.log 2>&1; cat gpurun_out/s4_ab_flat512b.log
bash tools/ab_libs_n.sh 256 noflat > gpurun_out/s4_ab_flat256.log 2>&1; cat gpurun_out/s4_ab_flat256.log
