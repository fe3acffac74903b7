timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python bench.py --latency --steps 200 --warmup 10 > gpurun_out/bench_latency.json 2>&1; tail -c 900 gpurun_out/bench_latency.json
python bench.py --keyswitch --steps 10 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read())['results']; print({k: round(v['ms'],3) for k,v in d.items()})"
