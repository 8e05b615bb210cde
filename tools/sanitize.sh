#!/bin/bash
# compute-sanitizer over every kernel family (tools/sanitize_cases.py);
# logs to gpurun_out/sanitize_<tool>.log.  Run under gpurun.
set -u
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 \
    --kernel-name regex:"conv_|splitk|s2d|unblock|im2col|weight" \
    python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -c 'ERROR SUMMARY' gpurun_out/sanitize_$tool.log) $(grep 'ERROR SUMMARY\|ALL OK\|MISMATCH' gpurun_out/sanitize_$tool.log | tr '\n' ' ')"
done
