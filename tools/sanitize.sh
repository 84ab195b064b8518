#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py (every product path at small n); summaries to gpurun_out/
cd "$(dirname "$0")/.."
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py \
    > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitizer_$tool.txt
done
