# suite-level tuner check: bench with and without --tune 2 on one box
for b in 256 32; do
  timeout 300 python bench.py --batch $b --no-e2e --no-cpu-baseline > gpurun_out/b${b}_def.json 2> gpurun_out/b${b}_def.err
  timeout 600 python bench.py --batch $b --no-e2e --no-cpu-baseline --tune 2 > gpurun_out/b${b}_tune.json 2> gpurun_out/b${b}_tune.err
done
timeout 300 python bench.py --profile f16 --batch 64 --no-e2e --no-cpu-baseline > gpurun_out/f16_def.json 2> gpurun_out/f16_def.err
timeout 600 python bench.py --profile f16 --batch 64 --no-e2e --no-cpu-baseline --tune 2 > gpurun_out/f16_tune.json 2> gpurun_out/f16_tune.err
for f in b256_def b256_tune b32_def b32_tune f16_def f16_tune; do python -c "import json,sys; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d['config'].get('tuned_plans'))" || tail -5 gpurun_out/$f.err; done
