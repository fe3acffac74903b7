timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for wl in cfg3 cfg4 cfg5; do python bench.py --workload $wl --steps 50 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$wl ms %.4f value %.4e frac %.3f'%(d['ms_per_step'], d['value'], d['roofline']['frac']))"; done
