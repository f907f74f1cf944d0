#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x tests/test_gpu_generic_n.py > gpurun_out/t_gen.log 2>&1; echo "rc=$?" >> gpurun_out/t_gen.log
python tools/generic_n_time.py 96 192 384 768 > gpurun_out/generic_t2.log 2>&1
