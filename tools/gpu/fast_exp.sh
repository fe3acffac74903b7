python bench.py --steps 50 --warmup 5 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('exact', [round(p['ms'],4) for p in d['parts']])"
cp paper_2410_05934_b200/librnsntt_fast.so paper_2410_05934_b200/librnsntt.so
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "all_sizes or cfg2 or cfg3 or edge or in_place" 2>&1 | tail -1
python bench.py --steps 50 --warmup 5 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fast', [round(p['ms'],4) for p in d['parts']])"
