timeout 850 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -1
for w in cfg3 cfg4 cfg5; do python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', 'ms %.4f'%d['ms_per_step'], [round(p['ms'],4) for p in d['parts']], 'e2e %.3e'%d['e2e']['value'])"; done
