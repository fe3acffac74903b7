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
# (11,2,1), (16,1,1), (12,1,2): cluster kernel; (13,5,1): limb split over streams; (16,2,2): three kernels
# (13,1,1), (15,1,1): k_clat with 16-CTA clusters; (10,1,520): the LZ warp engine (> 512 units)
for logn, limbs, batch in ((4, 2, 5), (7, 1, 3), (10, 2, 3), (11, 2, 1), (16, 1, 1), (12, 1, 2), (13, 5, 1),
                          (16, 2, 2), (13, 1, 1), (15, 1, 1), (10, 1, 520)):
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
# key switching: fused (one-prime digits) and unfused (two-prime digits) paths
for logn, L, K, dnum in ((11, 3, 1, 3), (11, 4, 2, 2)):
    n = 1 << logn
    mods = O.primes(logn, L + K)
    qs, pp = mods[:L], mods[L:]
    dd = inputs.residues(3, 1, qs, n)[0]
    evk = inputs.residues(4, 2 * dnum, mods, n).reshape(dnum, 2, L + K, n)
    a0 = inputs.residues(5, 1, qs, n)[0]
    ks = R.KeySwitch(R.Plan(logn, qs), R.Plan(logn, mods), dnum)
    out = torch.empty((2, L, n), dtype=torch.int64, device="cuda")
    ks(out, dev(dd), dev(evk), add0=dev(a0))
    ok &= np.array_equal(host(out), O.keyswitch(dd, evk, qs, pp, dnum, add0=a0))
# automorphism and BConv
ps = O.primes(11, 3)
p = R.Plan(11, ps)
a = inputs.residues(6, 2, ps, 1 << 11)
d = torch.empty(a.shape, dtype=torch.int64, device="cuda")
R.automorph(p, d, dev(a), 5, ntt_domain=False)
ok &= np.array_equal(host(d)[1, 2], O.automorph(a[1, 2], ps[2], 5))
pd = R.Plan(11, O.primes(11, 5)[3:])
bc = R.BConv(p, pd)
o2 = torch.empty((2, 2, 1 << 11), dtype=torch.int64, device="cuda")
bc(o2, dev(a))
ok &= np.array_equal(host(o2)[0], O.bconv(a[0], ps, O.primes(11, 5)[3:]))
# external product (CTA-parallel kernel), N = 2^10, l = 3
ps = O.primes(10, 1)
p = R.Plan(10, ps)
c = inputs.residues(7, 2 * 3, ps, 1 << 10).reshape(3, 2, 1 << 10)
z = inputs.residues(8, 2 * 3 * 2, ps, 1 << 10).reshape(6, 2, 1 << 10)
o3 = torch.empty(c.shape, dtype=torch.int64, device="cuda")
R.external_product(p, o3, dev(c), dev(z), 20, 3)
ok &= all(np.array_equal(host(o3)[s_], O.external_product(c[s_], z, ps[0], O.min_psi(ps[0], 10), 20, 3))
          for s_ in range(3))
# HRF-MatVec (f4), N = 2^12, 2 limbs, 5 slots, with the "+ b" term
ps = O.primes(12, 2)
p = R.Plan(12, ps)
pt = inputs.residues(9, 5, ps, 1 << 12)
ct = inputs.residues(10, 10, ps, 1 << 12).reshape(5, 2, 2, 1 << 12)
ad = inputs.residues(11, 2, ps, 1 << 12)
o4 = torch.empty((2, 2, 1 << 12), dtype=torch.int64, device="cuda")
R.hrf_matvec(p, o4, dev(pt), dev(ct), add=dev(ad))
ok &= np.array_equal(host(o4), O.hrf_matvec(pt, ct, ps, add=ad))
torch.cuda.synchronize()
print("sanitize run ok" if ok else "MISMATCH")
