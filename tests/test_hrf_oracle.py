"""Pins of the oracle's HRF-MatVec (tab:repack P:393-395).

oracle.hrf_matvec computes out[c][l] = add[c][l] + sum_j pt[j][l] (.) ct[j][c][l] in
the NTT domain.  It is pinned here against things other than itself:

* the convolution theorem: INTT(out_c) equals the sum of negacyclic
  products of the coefficient-form operands, computed with Python big integers
  by the schoolbook definition, plus INTT(add_c);
* decryption linearity of noiseless RLWE encryptions (the repack MatVec "As + b",
  P:358): for ct_j = (m_j - a_j s, a_j), out decrypts to sum_j p_j m_j + b;
* the special case n_slot = 1 without add, which is the pinned pointwise product;
* 60-bit primes (reading C2), several limbs, so a dropped 128-bit carry shows up.
"""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.filterwarnings("ignore")


def negacyclic(a, b, q):
    n = len(a)
    c = [0] * n
    for i in range(n):
        for j in range(n):
            k = i + j
            if k < n:
                c[k] += int(a[i]) * int(b[j])
            else:
                c[k - n] -= int(a[i]) * int(b[j])
    return [x % q for x in c]


def rand(rng, shape, qs, lim_axis):
    """uniform residues; limb index on axis lim_axis."""
    out = np.empty(shape, dtype=np.uint64)
    it = np.nditer(out, flags=["multi_index"], op_flags=["writeonly"])
    for x in it:
        q = qs[it.multi_index[lim_axis]]
        x[...] = int(rng.integers(0, q, dtype=np.uint64)) if q > 2**62 else int(rng.integers(0, q))
    return out


@pytest.mark.parametrize("logn,qs,ns", [(4, [97, 193], 5), (4, None, 3), (3, [17, 97, 113], 4)])
def test_hrf_matvec_convolution_theorem(logn, qs, ns):
    n = 1 << logn
    if qs is None:
        qs = O.primes(logn, 3)      # 60-bit
    psis = [O.min_psi(q, logn) for q in qs]
    L = len(qs)
    rng = np.random.default_rng(7 + logn + ns)
    p = rand(rng, (ns, L, n), qs, 1)          # plaintext diagonals, coefficient form
    c = rand(rng, (ns, 2, L, n), qs, 2)       # rotation ciphertexts, coefficient form
    b = rand(rng, (2, L, n), qs, 1)
    pt = np.stack([np.stack([O.ntt_fwd(p[j, l], qs[l], psis[l]) for l in range(L)]) for j in range(ns)])
    ct = np.stack([np.stack([np.stack([O.ntt_fwd(c[j, t, l], qs[l], psis[l]) for l in range(L)])
                             for t in range(2)]) for j in range(ns)])
    bh = np.stack([np.stack([O.ntt_fwd(b[t, l], qs[l], psis[l]) for l in range(L)]) for t in range(2)])
    out = O.hrf_matvec(pt, ct, qs, add=bh)
    out0 = O.hrf_matvec(pt, ct, qs)
    for t in range(2):
        for l in range(L):
            q = qs[l]
            want = [int(x) for x in b[t, l]]
            want0 = [0] * n
            for j in range(ns):
                prod = negacyclic(p[j, l], c[j, t, l], q)
                want = [(x + y) % q for x, y in zip(want, prod)]
                want0 = [(x + y) % q for x, y in zip(want0, prod)]
            assert [int(x) for x in O.ntt_inv(out[t, l], q, psis[l])] == want
            assert [int(x) for x in O.ntt_inv(out0[t, l], q, psis[l])] == want0


def test_hrf_matvec_decrypts_to_plaintext_sum():
    """Noiseless RLWE: ct_j = (m_j - a_j s, a_j); Dec(out) = out_0 + out_1 s = sum_j p_j m_j + b."""
    logn, ns = 4, 6
    n = 1 << logn
    qs = O.primes(logn, 2)
    psis = [O.min_psi(q, logn) for q in qs]
    rng = np.random.default_rng(11)
    for l, (q, psi) in enumerate(zip(qs, psis)):
        s = [int(x) for x in rng.integers(-1, 2, n)]
        s = [x % q for x in s]
        p = [[int(x) for x in rng.integers(0, q, n)] for _ in range(ns)]
        m = [[int(x) for x in rng.integers(0, q, n)] for _ in range(ns)]
        a = [[int(x) for x in rng.integers(0, q, n)] for _ in range(ns)]
        bb = [int(x) for x in rng.integers(0, q, n)]
        c0 = [[(mi - x) % q for mi, x in zip(m[j], negacyclic(a[j], s, q))] for j in range(ns)]
        F = lambda v: O.ntt_fwd(np.array(v, dtype=np.uint64), q, psi)   # noqa: E731
        pt = np.stack([F(p[j]) for j in range(ns)])[:, None, :]
        ct = np.stack([np.stack([F(c0[j]), F(a[j])]) for j in range(ns)])[:, :, None, :]
        add = np.stack([F(bb), np.zeros(n, dtype=np.uint64)])[:, None, :]
        out = O.hrf_matvec(pt, ct, [q], add=add)
        dec = O.ntt_inv(O.pointwise(out[1, 0], F(s), q), q, psi)
        dec = [(int(x) + int(y)) % q for x, y in zip(O.ntt_inv(out[0, 0], q, psi), dec)]
        want = bb[:]
        for j in range(ns):
            want = [(x + y) % q for x, y in zip(want, negacyclic(p[j], m[j], q))]
        assert dec == want


def test_hrf_matvec_single_slot_is_pointwise():
    qs = O.primes(5, 2)
    rng = np.random.default_rng(3)
    pt = np.stack([rng.integers(0, q, 32).astype(np.uint64) for q in qs])[None]
    ct = np.stack([np.stack([rng.integers(0, q, 32).astype(np.uint64) for q in qs]) for _ in range(2)])[None]
    out = O.hrf_matvec(pt, ct, qs)
    for t in range(2):
        for l, q in enumerate(qs):
            assert np.array_equal(out[t, l], O.pointwise(pt[0, l], ct[0, t, l], q))


def test_hrf_matvec_rejects_noncanonical():
    with pytest.raises(ValueError):
        O.hrf_matvec(np.full((1, 1, 4), 17, np.uint64), np.zeros((1, 2, 1, 4), np.uint64), [17])
