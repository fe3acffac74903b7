"""Seeded key material for the key-switching tests (f2; readings KS1-KS4).

Test infrastructure: builds noiseless switching keys with the oracle's
pinned transforms, evk_j = (-a_j s + P g_j s', a_j) in NTT form over QP, where
g_j = 1 mod the primes of digit j and 0 mod the other primes of Q (P g_j = 0
mod every prime of P).  No arithmetic of the key switch itself lives here.
"""
import numpy as np

import inputs
import oracle as O


def ternary(seed, n, weight):
    """Ternary polynomial with `weight` nonzero coefficients (as Python ints)."""
    rng = np.random.default_rng(seed)
    s = np.zeros(n, dtype=np.int64)
    idx = rng.choice(n, size=weight, replace=False)
    s[idx] = rng.choice([-1, 1], size=weight)
    return s


def ntt_of_small(s, moduli):
    """NTT form [len(moduli)][N] of a small signed integer polynomial."""
    return np.stack([O.ntt_fwd(np.array([int(c) % q for c in s], dtype=np.uint64), q, O.min_psi(q, len(s).bit_length() - 1))
                     for q in moduli])


def make_keys(logn, L, K, dnum, seed=7, weight=None):
    n = 1 << logn
    mods = O.primes(logn, L + K)
    qs, ps = mods[:L], mods[L:]
    weight = weight or max(1, n // 4)
    s = ternary(seed, n, weight)
    s2 = ternary(seed + 1, n, weight)
    S = ntt_of_small(s, mods)
    S2 = ntt_of_small(s2, mods)
    alpha = -(-L // dnum)
    P = 1
    for p in ps:
        P *= p
    evk = np.zeros((dnum, 2, L + K, n), dtype=np.uint64)
    a = inputs.residues(seed + 2, dnum, mods, n)          # uniform NTT-form a_j
    for j in range(dnum):
        for t, m in enumerate(mods):
            ajs = O.pointwise(a[j, t], S[t], m)
            b = (m - ajs) % m                              # -a_j s
            if t < L and j * alpha <= t < (j + 1) * alpha:
                pg = np.full(n, P % m, dtype=np.uint64)   # P g_j mod q_t = P mod q_t on digit j
                b = (b + O.pointwise(pg, S2[t], m)) % m
            evk[j, 0, t] = b
            evk[j, 1, t] = a[j, t]
    return dict(qs=qs, ps=ps, s=s, s2=s2, S=S, S2=S2, evk=evk, n=n, weight=weight)


def phase_error(out, d, keys):
    """Centered coefficients of INTT(out0 + out1 S - d S') per limb of Q, as a
    [L][N] int array (the key-switch error polynomial seen in every limb)."""
    qs = keys["qs"]
    L, n = d.shape
    errs = []
    for i, q in enumerate(qs):
        v = (out[0, i] + O.pointwise(out[1, i], keys["S"][i], q)) % q
        v = (v + q - O.pointwise(d[i], keys["S2"][i], q)) % q
        r = O.ntt_inv(v, q, O.min_psi(q, n.bit_length() - 1))
        errs.append([int(x) if int(x) <= q // 2 else int(x) - q for x in r])
    return np.array(errs, dtype=object)
