# full round-end style check: GPU tests, smoke, default bench (+e2e, cpu baseline), reference arm,
# batch-32 / fp16 lines, and the ncu launch list (plans fixed to defaults: --tune 0, see profiles/)
timeout 900 python -m pytest tests -m gpu -q -rf 2>&1 | tail -6 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python bench.py --batch 32 --no-e2e --no-cpu-baseline > gpurun_out/bench_b32.json 2> gpurun_out/bench_b32.err
timeout 600 python bench.py --profile f16 --batch 64 --no-e2e --no-cpu-baseline > gpurun_out/bench_f16.json 2> gpurun_out/bench_f16.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --tune 0 > gpurun_out/ncu_launch.log 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/smoke.log
for f in bench bench_ref bench_b32 bench_f16; do python -c "import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], d.get('ms_per_step'), (d.get('e2e') or {}).get('value'), d.get('clocks'))" || tail -3 gpurun_out/$f.err; done
