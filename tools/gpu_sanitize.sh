#!/bin/bash
# compute-sanitizer over the small stack workload: memcheck, racecheck (shared
# memory hazards), synccheck (barrier misuse).  Summaries -> gpurun_out/san_*.txt
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 300 python tools/sanitize_stack.py > gpurun_out/san_plain.txt 2>&1; echo "plain rc=$?" >> gpurun_out/san_plain.txt
for tool in memcheck racecheck synccheck; do
  timeout 900 $CS --tool $tool --print-limit 50 python tools/sanitize_stack.py > gpurun_out/san_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/san_$tool.txt
  tail -3 gpurun_out/san_$tool.txt
done
