for r in 1 2; do
for v in "--opt producers=1" "--opt producers=2"; do
  python bench.py --profile f16 --batch 64 --steps 20 --warmup 5 --no-e2e $v > gpurun_out/ab.json 2>gpurun_out/ab.err; python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('f16 $v', d['value'])"
  python bench.py --workload gemm4096 --steps 20 --warmup 5 --no-e2e $v > gpurun_out/ab.json 2>gpurun_out/ab.err; python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('gemm $v', d['value'])"
  python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline $v > gpurun_out/ab.json 2>gpurun_out/ab.err; python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('i8 $v', d['value'])"
done; done
