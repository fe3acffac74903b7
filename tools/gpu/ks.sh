# f2 key switch: bench line + per-kernel launch list of one paper-parameter key switch.
python bench.py --keyswitch --steps 20 --warmup 3 > gpurun_out/bench_keyswitch.json 2>gpurun_out/ks.err; cat gpurun_out/bench_keyswitch.json; tail -3 gpurun_out/ks.err
cat > /tmp/ks1.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import inputs, paper_2410_05934_b200 as R
from bench import primes_for
logn, L, K, dnum = 16, 45, 1, 45
n = 1 << logn
mods = primes_for(logn, L + K)
qp, qpp = R.Plan(logn, mods[:L]), R.Plan(logn, mods)
ks = R.KeySwitch(qp, qpp, dnum)
d = torch.from_numpy(inputs.residues(0, 1, mods[:L], n).view(np.int64)).cuda()
evk = torch.from_numpy(inputs.residues(1, 2 * dnum, mods, n).view(np.int64)).cuda()
out = torch.empty((2, L, n), dtype=torch.int64, device="cuda")
for _ in range(3):
    ks(out, d, evk)
torch.cuda.synchronize()
PY
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ks_launches.csv python /tmp/ks1.py > /dev/null 2>&1
