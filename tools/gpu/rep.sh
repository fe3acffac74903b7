nvidia-smi --query-gpu=clocks.sm,temperature.gpu,power.draw --format=csv
for i in 1 2 3; do python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5', round(d['ms_per_step'],4), round(d['roofline']['frac'],4), [(p['log2n'], round(p['ms'],4)) for p in d['parts']], d['clocks'])"; done
