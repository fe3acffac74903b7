"""Single-polynomial forward NTT launches for N = 2^12..2^16 (56-bit prime) -- run under ncu."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import inputs
import paper_2410_05934_b200 as R
from bench import primes_below

for logn in range(12, 17):
    q = primes_below(56, logn, 1)
    plan = R.Plan(logn, q)
    d = torch.from_numpy(inputs.residues(0, 1, q, 1 << logn).view(np.int64)).cuda()
    o = torch.empty_like(d)
    for _ in range(3):
        R.ntt_forward(plan, o, d)
    torch.cuda.synchronize()
