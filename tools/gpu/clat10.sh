set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cluster_path or latency_path or variants or edge or all_sizes" 2>&1 | tail -3
cat > /tmp/l10.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, ".")
import inputs, paper_2410_05934_b200 as R
from bench import primes_for
for logn in (10, 11):
    ps = primes_for(logn, 1); p = R.Plan(logn, ps)
    a = torch.from_numpy(inputs.residues(0, 1, ps, 1 << logn).view(np.int64)).cuda(); b = a.clone(); c = torch.empty_like(a)
    for _ in range(5): R.polymul(p, c, a, b, b_is_eval=True)
    g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(100): R.polymul(p, c, a, b, b_is_eval=True, stream=s)
    torch.cuda.synchronize(); g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): g.replay()
    e1.record(); torch.cuda.synchronize()
    print("polymul 2^%d single poly (graph): %.2f us" % (logn, e0.elapsed_time(e1) * 1e3 / 500))
PY
for v in 1 0; do echo "RNT_CLAT=$v"; RNT_CLAT=$v python /tmp/l10.py; done
for v in 1 0; do RNT_CLAT=$v python bench.py --workload cfg1 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('CLAT=$v cfg1', d['ms_per_step'], d['l2_warm']['ms_per_step'], d['parts'][0]['ms'])"; done
