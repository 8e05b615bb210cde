#!/bin/bash
# ncu --set full of the named suite layers (second launch of each captured too).
# usage: bash tools/ncu_full_layers.sh TAG layer [layer ...]
set -u
tag=$1; shift
mkdir -p gpurun_out
python tools/run_families.py "$@" > gpurun_out/${tag}_plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/${tag}_plain.log; exit 1; }
timeout 1800 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"conv_" \
  -o gpurun_out/${tag} -f python tools/run_families.py "$@" > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu rc=$?"
