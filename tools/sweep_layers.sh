#!/bin/bash
# Per-layer graph-replayed time for each option variant (one box), for picking shape rules.
# VARIANTS overrides the list (word-split: one variant per word group is not supported; edit the list).
# Table: python tools/sweep_table.py <output>
L="stem7x7 c2_1x1_64_64 c2_3x3_64 c2_1x1_64_256 c2_1x1_256_64 c3_1x1_256_128 c3_3x3s2_128 c3_1x1_128_512 c3_1x1s2_256_512 c3_1x1_512_128 c3_3x3_128 c4_1x1_512_256 c4_3x3s2_256 c4_1x1_256_1024 c4_1x1s2_512_1024 c4_1x1_1024_256 c4_3x3_256 c5_1x1_1024_512 c5_3x3s2_512 c5_1x1_512_2048 c5_1x1s2_1024_2048 c5_1x1_2048_512 c5_3x3_512"
for o in ${VARIANTS:-"" "--opt tma_store=1" "--opt l2_hints=0" "--opt l2_hints=3" "--opt st256=0" "--opt ws_epi_groups=2" "--opt b_res=1" "--opt ws_1x1=1"}; do
  echo "== $o"
  python tools/layer_timing.py $L $o 2>&1 | sed "s/{.eager.: [0-9.]*, .graph_events.: [0-9.]*, .graph_rep.: //; s/} us//"
done
