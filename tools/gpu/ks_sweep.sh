# Digit-split sweep of the fused key product + one ncu --set full capture of k_row_mac.
timeout 600 python -m pytest tests/test_gpu_keyswitch.py -q -x -m gpu 2>&1 | tail -1
RNT_KS_SPLIT=3 timeout 600 python -m pytest tests/test_gpu_keyswitch.py -q -x -m gpu -k "matches or paper" 2>&1 | tail -1
for sp in 1 2 3 5; do
  RNT_KS_SPLIT=$sp python bench.py --keyswitch --steps 10 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read())['results']; print('split $sp', {k: round(v['ms'],3) for k,v in d.items()})"
done
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
for _ in range(2):
    ks(out, d, evk)
torch.cuda.synchronize()
PY
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_row_mac -c 1 -o gpurun_out/ks_rowmac -f python /tmp/ks1.py > gpurun_out/ncu_ks.log 2>&1; tail -2 gpurun_out/ncu_ks.log
