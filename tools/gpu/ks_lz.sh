set -x
timeout 1200 python -m pytest tests/test_gpu_keyswitch.py -q -x 2>&1 | tail -3
for z in 1 0; do RNT_LAZY=$z python bench.py --keyswitch --steps 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('LAZY=$z', {k: round(v['ms'],3) for k,v in d['results'].items() if isinstance(v, dict) and 'ms' in v})"; done
python bench.py --keyswitch --steps 10 2>&1 | tail -1 > gpurun_out/bench_keyswitch.json
