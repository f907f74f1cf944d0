#!/bin/bash
mkdir -p gpurun_out
bash tools/ab_libs_n.sh 1024 r1tab > gpurun_out/ab_r1tab.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "multiprocess_peer_direct" > gpurun_out/t_mp1.log 2>&1; echo "rc=$?" >> gpurun_out/t_mp1.log
AB_LIB=$PWD/libsdns_nosplit.so timeout 600 python -m pytest tests -m gpu -q -x -k "multiprocess_peer_direct" > gpurun_out/t_mp2.log 2>&1; echo "rc=$?" >> gpurun_out/t_mp2.log
