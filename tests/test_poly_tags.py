"""RnsPoly domain / basis / plan tags.

CPU tests: the checks run on the host before any library call, so a stand-in
plan object and CPU tensors exercise every error path.  The GPU test runs the
tagged operations through the library against the oracle.
"""
from types import SimpleNamespace

import numpy as np
import pytest
import torch

import paper_2410_05934_b200 as R
from paper_2410_05934_b200 import poly as P


def fake_plan(logn=4, moduli=(97, 193)):
    return SimpleNamespace(log2n=logn, n_limbs=len(moduli), moduli=list(moduli))


def mk(plan, domain=P.COEFF, batch=1):
    return P.RnsPoly(torch.zeros(batch, plan.n_limbs, 1 << plan.log2n, dtype=torch.int64), plan, domain)


def test_shape_checked_against_plan():
    pl = fake_plan()
    with pytest.raises(P.PlanMismatch):
        P.RnsPoly(torch.zeros(3, 16, dtype=torch.int64), pl)       # 48 elements, not k * 2 * 16
    with pytest.raises(ValueError):
        P.RnsPoly(torch.zeros(2, 16, dtype=torch.int64), pl, "time")
    a = mk(pl, batch=3)
    assert a.batch == 3 and a.n == 16 and a.moduli == (97, 193)


def test_forward_needs_coeff_inverse_needs_eval():
    pl = fake_plan()
    with pytest.raises(P.DomainMismatch):
        P.forward(mk(pl, P.EVAL))
    with pytest.raises(P.DomainMismatch):
        P.inverse(mk(pl, P.COEFF))


def test_plan_mismatch_on_n_and_basis():
    pl = fake_plan()
    with pytest.raises(P.PlanMismatch):
        P.forward(mk(pl), plan=fake_plan(logn=5))
    with pytest.raises(P.BasisMismatch):
        P.forward(mk(pl), plan=fake_plan(moduli=(97, 257)))


def test_pointwise_rules():
    pl = fake_plan()
    with pytest.raises(P.DomainMismatch):
        P.pointwise_mul(mk(pl, P.EVAL), mk(pl, P.COEFF))
    with pytest.raises(P.DomainMismatch):
        P.pointwise_mul(mk(pl, P.COEFF), mk(pl, P.EVAL))
    with pytest.raises(P.BasisMismatch):
        P.pointwise_mul(mk(pl, P.EVAL), mk(fake_plan(moduli=(97, 257)), P.EVAL))
    with pytest.raises(P.PlanMismatch):
        P.pointwise_mul(mk(pl, P.EVAL), mk(fake_plan(logn=5), P.EVAL))
    with pytest.raises(ValueError):
        P.pointwise_mul(mk(pl, P.EVAL, batch=3), mk(pl, P.EVAL, batch=2))


def test_polymul_and_automorph_rules():
    pl = fake_plan()
    with pytest.raises(P.DomainMismatch):
        P.polymul(mk(pl, P.EVAL), mk(pl))
    with pytest.raises(P.BasisMismatch):
        P.polymul(mk(pl), mk(fake_plan(moduli=(193, 97))))       # same primes, other order
    with pytest.raises(ValueError):
        P.automorph(mk(pl), 4)


def test_package_exports():
    for name in ("RnsPoly", "COEFF", "EVAL", "DomainMismatch", "BasisMismatch", "PlanMismatch"):
        assert name in R.__all__ and hasattr(R, name)
    assert issubclass(R.DomainMismatch, ValueError)


@pytest.mark.gpu
@pytest.mark.parametrize("logn,limbs,batch", [(10, 2, 5), (16, 3, 1), (12, 4, 2)])
def test_tagged_ops_match_oracle(logn, limbs, batch):
    import inputs
    import oracle as O
    from helpers import from_dev, params, to_dev

    ps, psi = params(logn, limbs)
    pl = R.Plan(logn, ps)
    n = 1 << logn
    a_np = inputs.residues(31, batch, ps, n)
    b_np = inputs.residues(32, 1, ps, n)
    a = R.RnsPoly(to_dev(a_np), pl)
    b = R.RnsPoly(to_dev(b_np), pl)
    A = P.forward(a)
    assert A.domain == P.EVAL
    assert np.array_equal(from_dev(A.data), O.batch(O.OP_FWD, a_np, ps, psi, n_threads=8))
    B = P.forward(b)
    C = P.pointwise_mul(A, B)                                      # b broadcast over the batch
    c = P.inverse(C)
    want = O.batch(O.OP_POLYMUL, a_np, ps, psi, b=b_np, b_broadcast=True, n_threads=8)
    assert c.domain == P.COEFF and np.array_equal(from_dev(c.data), want)
    assert np.array_equal(from_dev(P.polymul(a, b).data), want)     # coefficient-form b
    assert np.array_equal(from_dev(P.polymul(a, B).data), want)     # Eval-form b (reading C8)
    g = 5
    s = P.automorph(A, g)
    assert s.domain == P.EVAL
    want_s = np.stack([np.stack([O.automorph(a_np[i, l], ps[l], g) for l in range(limbs)]) for i in range(batch)])
    assert np.array_equal(from_dev(P.inverse(s).data), want_s)
