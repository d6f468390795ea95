#!/bin/bash
# compute-sanitizer runs of tools/sanitize_driver.py; logs -> gpurun_out/
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $tool --print-limit 50 --target-processes all \
    python tools/sanitize_driver.py > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitizer_$tool.txt
  tail -n 3 gpurun_out/sanitizer_$tool.txt
done
