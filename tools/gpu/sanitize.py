"""Small invocations of every kernel family for compute-sanitizer (memcheck,
racecheck, synccheck, initcheck).  Checks results against the oracle too."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import inputs  # noqa: E402
import oracle as O  # noqa: E402
import paper_2410_05934_b200 as R  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64).copy()).cuda()


def host(t):
    return t.cpu().numpy().view(np.uint64)


ok = True
for logn, limbs, batch in ((4, 2, 5), (7, 1, 3), (10, 2, 3), (11, 2, 1), (16, 2, 2)):
    ps = O.primes(logn, limbs)
    psi = [O.min_psi(q, logn) for q in ps]
    p = R.Plan(logn, ps)
    a = inputs.residues(1, batch, ps, 1 << logn)
    b = inputs.residues(2, batch, ps, 1 << logn)
    bh = O.batch(O.OP_FWD, b, ps, psi)
    d = torch.empty(a.shape, dtype=torch.int64, device="cuda")
    R.ntt_forward(p, d, dev(a))
    ok &= np.array_equal(host(d), bh * 0 + O.batch(O.OP_FWD, a, ps, psi))
    R.ntt_inverse(p, d, dev(bh))
    ok &= np.array_equal(host(d), b)
    R.polymul(p, d, dev(a), dev(bh), b_is_eval=True)
    want = O.batch(O.OP_POLYMUL_EVAL, a, ps, psi, b=bh)
    ok &= np.array_equal(host(d), want)
    R.polymul(p, d, dev(a), dev(b))
    ok &= np.array_equal(host(d), want)
    R.pointwise_mul(p, d, dev(a), dev(b))
    torch.cuda.synchronize()
print("sanitize run ok" if ok else "MISMATCH")
