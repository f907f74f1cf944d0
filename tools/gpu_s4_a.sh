#!/bin/bash
# session baseline: full GPU suite with durations, then the default bench line
mkdir -p gpurun_out
( time timeout 1500 python -m pytest tests -m gpu -q -x --durations=25 ) > gpurun_out/s4_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s4_tests.log
( time timeout 900 python bench.py ) > gpurun_out/s4_bench.json 2> gpurun_out/s4_bench.err; echo "bench rc=$?"
tail -5 gpurun_out/s4_tests.log
