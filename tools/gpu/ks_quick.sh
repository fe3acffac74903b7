timeout 600 python -m pytest tests/test_gpu_keyswitch.py -q -x -m gpu 2>&1 | tail -1
python bench.py --keyswitch --steps 10 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read())['results']; print({k: round(v['ms'],3) for k,v in d.items()})"
