#!/bin/bash
# Checks of every kernel family on small shapes (tools/sanitize_cases.py):
#  1. the instrumented build (libtzc_b200_checks.so, `make -C paper_2101_08458_b200 checks`):
#     every mbarrier wait has a watchdog that prints and traps on a deadlock,
#     every epilogue global store is bounds-checked against the output /
#     split-K workspace extents; each case is also compared with the oracle;
#  2. compute-sanitizer memcheck/racecheck/synccheck/initcheck when the pool
#     allows it (it reports itself closed on this pool; the log says so).
set -u
mkdir -p gpurun_out
TZC_B200_CHECKS=1 timeout 900 python tools/sanitize_cases.py > gpurun_out/checks_build.log 2>&1
echo "instrumented build rc=$? $(grep -c 'OK$' gpurun_out/checks_build.log) OK, $(grep -c 'MISMATCH\|watchdog\|bounds' gpurun_out/checks_build.log) failures"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 \
    --kernel-name regex:"conv_|splitk|s2d|stem|unblock|im2col|weight" \
    python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(head -c 300 gpurun_out/sanitize_$tool.log | head -2 | tr '\n' ' ')"
done
