#!/bin/bash
# A/B the bench on one box: alternate variants (each "--opt a=b --opt c=d" or "")
# for R rounds; print value per run.  usage: bash tools/ab_bench.sh R "variant1" "variant2" ...
R=$1; shift
for r in $(seq 1 $R); do
  for v in "$@"; do
    python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline $v > gpurun_out/ab.json 2> gpurun_out/ab.err
    python - "$v" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
print(f"{sys.argv[1] or 'default':40s} {d['value']:8.1f} TOPS  {d['ms_per_step']*1000:7.1f} us")
PY
  done
done
