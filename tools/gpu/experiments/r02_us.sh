# U/S scaled-twiddle inverse: parity + bench
O=gpurun_out/us; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt
for i in 1 2; do python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-graph > $O/cfg5_$i.json 2>&1; echo "cfg5 $(tail -1 $O/cfg5_$i.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],5), [round(p["ms"],5) for p in d["parts"]], round(d["roofline"]["frac"],4), d["digests_ok"])')"; done
python bench.py --workload cfg2 --steps 50 --no-cpu-baseline --no-e2e --no-graph > $O/cfg2.json 2>&1; echo "cfg2 $(tail -1 $O/cfg2.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],5), round(d["roofline"]["frac"],4), d["digests_ok"])')"
python bench.py --extprod --steps 20 > $O/ext.json 2>&1; tail -1 $O/ext.json | head -c 600; echo
