timeout 1700 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for wl in cfg1 cfg5; do python bench.py --workload $wl --steps 50 --warmup 5 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$wl ms %.4f value %.4e e2e %.4e frac %.3f launches %d'%(d['ms_per_step'], d['value'], d['e2e']['value'], d['roofline']['frac'], d['gpu_launches']))"; done
