# LZ (lazy CT ranges) vs Harvey: parity + bench A/B
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "lazy or variants or cfg5 or cfg2 or cfg3 or cfg4 or edge or all_sizes or split or chunk" 2>&1 | tail -3
for z in 1 0 1 0; do RNT_LAZY=$z python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('LAZY=$z cfg5', d['ms_per_step'], [ (p['log2n'], round(p['ms'],4), round(p['frac_alu'],3)) for p in d['parts']])"; done
for z in 1 0; do RNT_LAZY=$z python bench.py --workload cfg2 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('LAZY=$z cfg2', d['ms_per_step'], d['roofline']['frac'])"; done
for z in 1 0; do for w in cfg3 cfg4; do RNT_LAZY=$z python bench.py --workload $w --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('LAZY=$z $w', d['ms_per_step'], d['roofline']['frac'])"; done; done
