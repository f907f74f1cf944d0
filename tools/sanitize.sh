#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over
# tools/sanitize_case.py (n = 16 and 32, p = 1, slab 2, pencil 2x2). Logs and
# one-line summaries go to gpurun_out/sanitize/.
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  timeout 1500 $CS --tool $tool $extra --print-limit 50 --target-processes all \
    python tools/sanitize_case.py > gpurun_out/sanitize/$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize/$tool.log | tail -1)" \
    >> gpurun_out/sanitize/summary.txt
done
