#!/bin/bash
python tools/pair_probe.py > gpurun_out/pair_plain.log 2>&1 || { tail gpurun_out/pair_plain.log; exit 1; }
/usr/local/cuda/bin/ncu --clock-control none -k regex:"conv_tc" --csv \
  --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,l1tex__m_xbar2l1tex_read_bytes.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__cluster_dim_x \
  python tools/pair_probe.py > gpurun_out/pair_ncu.csv 2> gpurun_out/pair_ncu.err
python - <<'PY'
import csv
rows=[l for l in open("gpurun_out/pair_ncu.csv") if l.startswith('"')]
r=list(csv.DictReader(rows))
from collections import OrderedDict
by=OrderedDict()
for x in r:
    key=(x["ID"], x["Kernel Name"].split("(")[0][:60])
    by.setdefault(key,{})[x["Metric Name"]]=x["Metric Value"]+" "+x["Metric Unit"]
for k,v in by.items():
    print(k[0], k[1], "|", " | ".join(f"{m.split('.')[0]}={val}" for m,val in v.items()))
PY
