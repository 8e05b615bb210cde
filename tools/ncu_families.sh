#!/bin/bash
# ncu --set full of every kernel family (tools/run_families.py), after a plain
# run exits 0.  Second launch of each layer is the captured one (-s skips the
# first launch of each pair is not possible per kernel; both are captured).
set -u
mkdir -p gpurun_out
python tools/run_families.py > gpurun_out/families_plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/families_plain.log; exit 1; }
timeout 2400 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on \
  -k regex:"conv_|splitk|s2d" -o gpurun_out/prof_r02_families -f python tools/run_families.py > gpurun_out/families_ncu.log 2>&1
echo "ncu rc=$?"
/usr/local/cuda/bin/ncu -i gpurun_out/prof_r02_families.ncu-rep --page raw --csv > gpurun_out/prof_r02_families_raw.csv 2>/dev/null
python tools/ncu_table.py gpurun_out/prof_r02_families_raw.csv > gpurun_out/prof_r02_families_table.md
rm -f gpurun_out/prof_r02_families.ncu-rep  # keep the CSV (the report is tens of MB)
head -40 gpurun_out/prof_r02_families_table.md
