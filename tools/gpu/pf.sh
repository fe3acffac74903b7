set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "lazy or variants or cfg5 or cfg2 or edge" 2>&1 | tail -2
for i in 1 2; do for v in 1 0; do for w in cfg5 cfg2; do RNT_PREFETCH=$v python bench.py --workload $w --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('PF=$v $w', round(d['ms_per_step'],4), round(d['roofline']['frac'],4), [(p['log2n'], round(p['ms'],4)) for p in d['parts']])"; done; done; done
