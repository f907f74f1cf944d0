#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/dbg_p1single.py 3 > gpurun_out/s4_dbg.log 2>&1; echo "dbg rc=$?"
( time timeout 1500 python -m pytest tests -m gpu -q --durations=15 --deselect tests/test_gpu_parity.py::test_p1_single_transform_items ) > gpurun_out/s4_tests2.log 2>&1; echo "tests rc=$?" >> gpurun_out/s4_tests2.log
tail -4 gpurun_out/s4_tests2.log
