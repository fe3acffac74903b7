timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "latency_path or variants or edge or all_sizes or in_place" 2>&1 | tail -2
for u in 0 8; do for wl in cfg1; do RNT_LAT_UNITS=$u python bench.py --workload $wl --steps 50 --warmup 5 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('lat$u $wl ms %.4f value %.4e e2e %.4e'%(d['ms_per_step'], d['value'], d['e2e']['value']))"; done; done
cat > /tmp/lat_sweep.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, ".")
import inputs, paper_2410_05934_b200 as R
from bench import primes_for
ps = primes_for(10, 1); p = R.Plan(10, ps)
for units in (1, 8, 64, 296, 512, 1024, 2048):
    a = torch.from_numpy(inputs.residues(0, units, ps, 1024).view(np.int64)).cuda(); b = a.clone(); c = torch.empty_like(a)
    for _ in range(5): R.polymul(p, c, a, b, b_is_eval=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(100): R.polymul(p, c, a, b, b_is_eval=True)
    e1.record(); torch.cuda.synchronize()
    print(units, round(e0.elapsed_time(e1) * 10, 2), "us per call")
PY
for u in 0 100000; do echo "RNT_LAT_UNITS=$u"; RNT_LAT_UNITS=$u python /tmp/lat_sweep.py; done
