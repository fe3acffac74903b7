set -x
timeout 900 python -m pytest tests/test_bench_contract.py tests/test_gpu_parity.py -q -x -k "contract or our_arm or cfg5" 2>&1 | tail -2
python bench.py 2>&1 | tail -1 > gpurun_out/bench_cfg5.json
python -c "import json; d=json.load(open('gpurun_out/bench_cfg5.json')); print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['parts_schedule'][:20], [(p['log2n'], round(p['ms'],4)) for p in d['parts']], d['e2e']['value'], d['clocks'])"
python bench.py --sequential-parts --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('seq', d['ms_per_step'], d['roofline']['frac'])"
for w in cfg2 cfg3; do python bench.py --workload $w --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['ms_per_step'], d['roofline']['frac'], d['parts_schedule'])"; done
