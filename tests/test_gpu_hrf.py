"""GPU parity of HRF-MatVec (tab:repack P:393-395):
rnt_hrf_matvec through the C ABI against oracle.hrf_matvec, bit-exact on every
element, at the bench shape (N = 2^16, 4 limbs), small and ragged shapes,
n_slot = 0, in-place accumulation, all-(q-1) inputs (the 192-bit accumulator's
top word) and moduli just below 2^62 (reading C5's upper limit)."""
import numpy as np
import pytest

import inputs
import oracle as O
from helpers import empty_dev, from_dev, params, to_dev

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2410_05934_b200 as R  # noqa: E402


def _operands(seed, n_slot, ps, n):
    pt = inputs.residues(seed, n_slot, ps, n)
    ct = inputs.residues(seed + 1, 2 * n_slot, ps, n).reshape(n_slot, 2, len(ps), n)
    add = inputs.residues(seed + 2, 2, ps, n)
    return pt, ct, add


@pytest.mark.parametrize("logn,L,n_slot", [(16, 4, 64), (16, 1, 257), (10, 3, 37), (4, 2, 5), (12, 2, 1),
                                           (13, 5, 9), (5, 1, 1024)])
def test_hrf_matvec_parity(logn, L, n_slot):
    ps, _ = params(logn, L)
    n = 1 << logn
    p = R.Plan(logn, ps)
    pt, ct, add = _operands(40 + logn, n_slot, ps, n)
    out = empty_dev((2, L, n))
    R.hrf_matvec(p, out, to_dev(pt), to_dev(ct), add=to_dev(add))
    assert np.array_equal(from_dev(out), O.hrf_matvec(pt, ct, ps, add=add))
    R.hrf_matvec(p, out, to_dev(pt), to_dev(ct))
    assert np.array_equal(from_dev(out), O.hrf_matvec(pt, ct, ps))


def test_hrf_matvec_in_place_accumulate_and_empty():
    logn, L = 11, 2
    ps, _ = params(logn, L)
    n = 1 << logn
    p = R.Plan(logn, ps)
    pt, ct, add = _operands(7, 33, ps, n)
    acc = to_dev(add)
    R.hrf_matvec(p, acc, to_dev(pt[:20]), to_dev(ct[:20]), add=acc)      # acc += first 20 terms
    R.hrf_matvec(p, acc, to_dev(pt[20:]), to_dev(ct[20:]), add=acc)      # acc += the rest
    assert np.array_equal(from_dev(acc), O.hrf_matvec(pt, ct, ps, add=add))
    out = empty_dev((2, L, n))
    R.hrf_matvec(p, out, None, None, n_slot=0, add=to_dev(add))         # n_slot = 0: out = add
    assert np.array_equal(from_dev(out), add)
    R.hrf_matvec(p, out, None, None, n_slot=0)                           # out = 0
    assert not from_dev(out).any()


def _primes_below_2_62(logn, count):
    two_n = 2 << logn
    k, out = ((1 << 62) - 1) // two_n, []
    while len(out) < count:
        q = k * two_n + 1
        if O.is_prime(q):
            out.append(q)
        k -= 1
    return out


@pytest.mark.parametrize("top", [False, True])
def test_hrf_matvec_extreme_values(top):
    """All operands q - 1: every product is (q-1)^2 ~ 2^120 (2^124 for 62-bit q), so
    the sum's top word is non-zero and the final reduction sees its largest inputs."""
    logn, n_slot = 12, 1100
    ps = _primes_below_2_62(logn, 2) if top else list(params(logn, 2)[0])
    n = 1 << logn
    p = R.Plan(logn, ps)
    pt = np.stack([np.full(n, q - 1, dtype=np.uint64) for q in ps])[None].repeat(n_slot, 0)
    ct = pt[:, None].repeat(2, 1)
    add = np.stack([np.full(n, q - 1, dtype=np.uint64) for q in ps])[None].repeat(2, 0)
    out = empty_dev((2, 2, n))
    R.hrf_matvec(p, out, to_dev(pt), to_dev(ct), add=to_dev(add))
    want = O.hrf_matvec(pt, ct, ps, add=add)
    assert np.array_equal(from_dev(out), want)
    for l, q in enumerate(ps):   # closed form: n_slot (q-1)^2 + (q-1) = n_slot - 1 mod q
        assert int(want[0, l, 0]) == (n_slot - 1) % q


def test_hrf_matvec_argument_errors():
    logn, L = 10, 2
    ps, _ = params(logn, L)
    n = 1 << logn
    p = R.Plan(logn, ps)
    pt, ct, _ = _operands(3, 4, ps, n)
    dpt, dct = to_dev(pt), to_dev(ct)
    with pytest.raises(ValueError):                                    # binding: out too small
        R.hrf_matvec(p, empty_dev((1, L, n)), dpt, dct)
    with pytest.raises(ValueError):                                    # binding: ct too small
        R.hrf_matvec(p, empty_dev((2, L, n)), dpt, dct[:3])
    with pytest.raises(R.RntError):                                    # C ABI: out overlaps ct
        R.hrf_matvec(p, dct, dpt, dct, n_slot=1)
    with pytest.raises(R.RntError):                                    # C ABI: unaligned out
        R.rnt_hrf_matvec(p, empty_dev((2 * L * n + 2,)).data_ptr() + 8, dpt, dct, n_slot=4)
