#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q tests/test_gpu_generic_n.py tests/test_gpu_multiprocess.py \
  "tests/test_gpu_parity.py::test_config_errors" "tests/test_gpu_runner.py::test_bench_rows_and_csv" \
  > gpurun_out/t2.log 2>&1; echo "t2 rc=$?" >> gpurun_out/t2.log
timeout 600 python bench.py --gpus 2 --transport host --n 256 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b2.log 2>&1; echo "b2 rc=$?" >> gpurun_out/b2.log
timeout 1800 bash tools/sanitize.sh
