#!/bin/bash
# Per-layer kernel table of the batch-256 int8 suite (every layer launched twice,
# tools/run_families.py suite) with a handful of ncu counters: duration, DRAM
# bytes, tensor-pipe and issue activity.  Cold caches (ncu default), clocks as set.
set -u
mkdir -p gpurun_out
tag=${1:-layers}
python tools/run_families.py suite > gpurun_out/${tag}_plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/${tag}_plain.log; exit 1; }
timeout 1200 /usr/local/cuda/bin/ncu --clock-control none -k regex:"conv_|splitk|s2d" \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_issued.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum \
  --csv python tools/run_families.py suite > gpurun_out/${tag}_ncu.csv 2> gpurun_out/${tag}_ncu.err
echo "ncu rc=$?"
python tools/ncu_layers_table.py gpurun_out/${tag}_ncu.csv gpurun_out/${tag}_plain.log > gpurun_out/${tag}_table.md
cat gpurun_out/${tag}_table.md
