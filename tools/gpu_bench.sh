# bench lines only: default (b256, e2e + cpu baseline), batch 32, fp16 batch 64
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --batch 32 --no-e2e --no-cpu-baseline > gpurun_out/bench_b32.json 2> gpurun_out/bench_b32.err
timeout 600 python bench.py --profile f16 --batch 64 --no-e2e --no-cpu-baseline > gpurun_out/bench_f16.json 2> gpurun_out/bench_f16.err
for f in bench bench_b32 bench_f16; do python -c "import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], d.get('ms_per_step'), (d.get('e2e') or {}).get('value'), d.get('clocks'), d['config'].get('plan_search'), d['config'].get('branch_assignment'))" || tail -3 gpurun_out/$f.err; done
