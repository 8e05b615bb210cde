#!/bin/bash
# Round-2 closing measurements on one box: the bench lines of every config,
# the reference arm, the per-layer ncu table (+ traffic.json source) and the
# ncu launch list of the headline command.  Outputs under gpurun_out/final/.
set -u
out=gpurun_out/final
mkdir -p $out
run() { local name=$1; shift; python bench.py "$@" > $out/$name.json 2> $out/$name.err; echo "$name rc=$? $(tail -c 300 $out/$name.json | head -c 200)"; }
run bench --steps 30 --warmup 5
run bench_b32 --batch 32 --steps 30 --warmup 5
run bench_f16 --profile f16 --batch 64 --steps 30 --warmup 5
run bench_gemm4096 --workload gemm4096 --steps 20 --warmup 5
run bench_c1 --workload c1 --steps 50 --warmup 5
run bench_ref --impl reference --steps 3 --warmup 3
bash tools/ncu_layers.sh final_layers > /dev/null 2>&1
cp gpurun_out/final_layers_* $out/ 2>/dev/null
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $out/launch_plain.log 2>&1 && \
  timeout 1200 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $out/launches_bench.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $out/launch_ncu.log 2>&1
echo "launch list rc=$?"
