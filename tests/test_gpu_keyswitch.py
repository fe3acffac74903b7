"""GPU parity of rnt_keyswitch_apply (f2) against the oracle's key switching.

Bit-exact on every output residue, from tiny shapes (several digits, K > 1,
ragged last digit) up to the paper's (N, L, dnum) = (2^16, 44 + 1, 45)
parameters with one special prime (reading KS1).
"""
import numpy as np
import pytest

import inputs
import oracle as O
import paper_2410_05934_b200 as R
from helpers import from_dev, to_dev, empty_dev

pytestmark = pytest.mark.gpu


def run_case(logn, L, K, dnum, seed=3, with_add0=False):
    n = 1 << logn
    mods = O.primes(logn, L + K)
    qs, ps = mods[:L], mods[L:]
    d = inputs.residues(seed, 1, qs, n)[0]
    evk = inputs.residues(seed + 1, dnum * 2, mods, n).reshape(dnum, 2, L + K, n)
    add0 = inputs.residues(seed + 2, 1, qs, n)[0] if with_add0 else None
    want = O.keyswitch(d, evk, qs, ps, dnum, add0=add0)
    qp, qpp = R.Plan(logn, qs), R.Plan(logn, mods)
    ks = R.KeySwitch(qp, qpp, dnum)
    out = empty_dev((2, L, n))
    ks(out, to_dev(d), to_dev(evk), to_dev(add0) if add0 is not None else None)
    got = from_dev(out)
    assert np.array_equal(got, want)
    return ks


# alpha = 1 with N >= 2^11 takes the fused path (lift in the column pass, key
# product in the row pass); the others the unfused ModUp / NTT / MAC kernels.
@pytest.mark.parametrize("logn,L,K,dnum", [(4, 3, 1, 3), (10, 4, 1, 4), (10, 5, 2, 2), (11, 6, 3, 3),
                                           (12, 7, 2, 3), (13, 3, 1, 1), (16, 4, 2, 2),
                                           (11, 4, 1, 4), (12, 3, 2, 3), (13, 5, 1, 5), (14, 2, 3, 2),
                                           (15, 3, 1, 3), (16, 6, 2, 6)])
def test_keyswitch_matches_oracle(logn, L, K, dnum):
    run_case(logn, L, K, dnum)


def test_keyswitch_add0():
    run_case(12, 4, 1, 4, with_add0=True)


@pytest.mark.slow
def test_keyswitch_paper_parameters():
    """(N, L + 1, dnum) = (2^16, 45, 45) with one special prime (KS1)."""
    ks = run_case(16, 45, 1, 45)
    assert ks.alpha == 1


def test_keyswitch_noiseless_key_relation():
    """Real key from the oracle-built key material: out0 + out1 s = d s' + small."""
    from keyswitch_keys import make_keys, phase_error

    logn, L, K, dnum = 10, 4, 2, 2
    keys = make_keys(logn, L, K, dnum)
    d = inputs.residues(11, 1, keys["qs"], keys["n"])[0]
    qp, qpp = R.Plan(logn, keys["qs"]), R.Plan(logn, keys["qs"] + keys["ps"])
    ks = R.KeySwitch(qp, qpp, dnum)
    out = empty_dev((2, L, keys["n"]))
    ks(out, to_dev(d), to_dev(keys["evk"]))
    e = phase_error(from_dev(out), d, keys)
    assert all((e[i] == e[0]).all() for i in range(L))
    assert max(abs(int(v)) for v in e[0]) < (1 + keys["weight"]) * (1 + K)


def test_keyswitch_argument_errors():
    logn = 10
    mods = O.primes(logn, 5)
    q, qp = R.Plan(logn, mods[:4]), R.Plan(logn, mods)
    for bad in (0, 5):
        with pytest.raises(R.RntError):
            R.KeySwitch(q, qp, bad)
    with pytest.raises(R.RntError):
        R.KeySwitch(qp, q, 2)                                  # P empty / swapped
    with pytest.raises(R.RntError):
        R.KeySwitch(R.Plan(logn, mods[1:5]), qp, 2)           # Q not a prefix of QP
    with pytest.raises(R.RntError):
        R.KeySwitch(q, qp, 3)                                  # alpha 2: (3-1)*2 >= 4 -> empty digit


UNFUSED_SCRIPT = r"""
import sys
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
from test_gpu_keyswitch import run_case
run_case(16, 6, 2, 6); run_case(12, 5, 1, 5, with_add0=True)
print("UNFUSED_OK")
"""


def test_keyswitch_unfused_variant():
    """RNT_KS_UNFUSED=1 forces the unfused kernels for one-prime digits too."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = UNFUSED_SCRIPT.format(root=root, tests=os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, "RNT_KS_UNFUSED": "1"}, capture_output=True,
                       text=True, timeout=600)
    assert "UNFUSED_OK" in r.stdout, r.stdout + r.stderr
