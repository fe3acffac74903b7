"""One key switch at the paper's parameters (2^16, 45 + 1 limbs, dnum 45), three times -- for ncu."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import inputs
import paper_2410_05934_b200 as R
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
