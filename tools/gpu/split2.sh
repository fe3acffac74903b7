set -x
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 2>&1 | tail -2
for w in cfg5 cfg2; do python bench.py --workload $w --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', round(d['ms_per_step'],4), round(d['roofline']['frac'],4), [(p['log2n'], round(p['ms'],4)) for p in d['parts']])"; done
python bench.py --extprod --steps 20 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: (round(v['ms'],4), round(v['frac_alu'],3)) for k,v in d['results'].items()})"
