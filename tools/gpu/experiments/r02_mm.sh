O=gpurun_out/mm; mkdir -p $O
for i in 1 2; do python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $O/bench_cfg5_$i.json 2>&1; done
python bench.py --workload cfg2 --steps 50 --no-cpu-baseline --no-e2e > $O/bench_cfg2.json 2>&1
python bench.py --workload cfg4 --steps 20 --no-cpu-baseline --no-e2e > $O/bench_cfg4.json 2>&1
python bench.py --keyswitch --steps 10 > $O/bench_keyswitch.json 2>&1
python bench.py --automorph --steps 20 > $O/bench_automorph.json 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest.txt 2>&1; tail -2 $O/pytest.txt
for f in $O/bench_*.json; do echo $f; tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d.get('value'), d.get('ms_per_step'), (d.get('roofline') or {}).get('frac'), str(d.get('results', ''))[:300])"; done
