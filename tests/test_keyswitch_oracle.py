"""Pins of the oracle's CKKS hybrid key switching (f2; readings KS1-KS4).

Against mathematics, not against itself: with a noiseless key
evk_j = (-a_j s + P g_j s', a_j), every correct key switch satisfies
    out0 + out1 s = d s' + e  (mod each q_i)
with one small integer polynomial e (the ModDown rounding plus, for K > 1,
the BConv overflow), |e_k| < (1 + h)(1 + K) for a ternary s of weight h.  A
dropped term, wrong sign, wrong digit or limb index, or a transposed
operand leaves e uniform mod q_i instead.
"""
import numpy as np
import pytest

import inputs
import oracle as O
from keyswitch_keys import make_keys, phase_error


@pytest.mark.parametrize("logn,L,K,dnum", [(4, 3, 1, 3), (4, 3, 1, 1), (5, 4, 2, 2), (6, 5, 2, 2), (5, 6, 3, 3),
                                           (4, 2, 1, 2)])
def test_keyswitch_relation(logn, L, K, dnum):
    keys = make_keys(logn, L, K, dnum)
    d = inputs.residues(11, 1, keys["qs"], keys["n"])[0]
    out = O.keyswitch(d, keys["evk"], keys["qs"], keys["ps"], dnum)
    e = phase_error(out, d, keys)
    assert all((e[i] == e[0]).all() for i in range(L)), "error polynomial differs between limbs"
    bound = (1 + keys["weight"]) * (1 + K)
    assert max(abs(int(v)) for v in e[0]) < bound


def test_keyswitch_broken_key_is_detected():
    """Sanity of the pin: a key for another secret leaves a uniform error."""
    logn, L, K, dnum = 4, 3, 1, 3
    keys = make_keys(logn, L, K, dnum)
    other = make_keys(logn, L, K, dnum, seed=99)
    d = inputs.residues(11, 1, keys["qs"], keys["n"])[0]
    out = O.keyswitch(d, other["evk"], keys["qs"], keys["ps"], dnum)
    e = phase_error(out, d, keys)
    assert max(abs(int(v)) for v in e[0]) > 2 ** 40


def test_keyswitch_zero_and_add0():
    logn, L, K, dnum = 5, 4, 1, 4
    keys = make_keys(logn, L, K, dnum)
    n = keys["n"]
    z = np.zeros((L, n), dtype=np.uint64)
    assert not O.keyswitch(z, keys["evk"], keys["qs"], keys["ps"], dnum).any()
    d = inputs.residues(12, 1, keys["qs"], n)[0]
    c0 = inputs.residues(13, 1, keys["qs"], n)[0]
    base = O.keyswitch(d, keys["evk"], keys["qs"], keys["ps"], dnum)
    withc = O.keyswitch(d, keys["evk"], keys["qs"], keys["ps"], dnum, add0=c0)
    assert np.array_equal(withc[1], base[1])
    for i, q in enumerate(keys["qs"]):
        assert np.array_equal(withc[0, i], (base[0, i] + c0[i]) % q)
