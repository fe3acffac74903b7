set -x
timeout 600 python -m pytest tests/test_bench_contract.py -q 2>&1 | tail -1
for i in 1 2; do
python bench.py --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('stream', d['value'], d['e2e'])"
python bench.py --no-cpu-baseline --e2e-serial 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('serial', d['value'], d['e2e']['value'])"
done
python bench.py --workload cfg4 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4', d['value'], d['e2e']['value'])"
