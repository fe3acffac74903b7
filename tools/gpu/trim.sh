set -x
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -2
python __graft_entry__.py --smoke 2>&1 | tail -1
python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5', round(d['ms_per_step'],4), d['value'], round(d['roofline']['frac'],4))"
python bench.py --latency 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: round(v['us_graph'],2) for k,v in d['results'].items()})"
