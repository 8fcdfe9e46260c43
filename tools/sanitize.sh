#!/bin/bash
# compute-sanitizer over tools/sanitize.py; logs to gpurun_out/sanitize_<tool>.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 50 \
    python tools/sanitize.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.log
done
