set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "external" 2>&1 | tail -2
for z in 1 0; do RNT_LAZY=$z python bench.py --extprod --steps 20 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('LAZY=$z', {k: (round(v['ms'],4), round(v['frac_alu'],3)) for k,v in d['results'].items()})"; done
python bench.py --extprod --steps 20 2>&1 | tail -1 > gpurun_out/bench_extprod.json
