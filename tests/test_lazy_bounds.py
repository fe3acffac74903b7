"""Range arithmetic of the kernels' lazy reductions (modarith.cuh),
checked with exact integers for the largest modulus each path accepts -- no GPU.

* LZ CT schedule (ct_bfly_lz, lz_bound_before): from canonical input the X bound grows by
  2q per stage and X is reduced by 8q only where the bound would pass 16q (stages 7, 11, 15);
  every intermediate must stay below 2^64, and the forward output must be a valid Montgomery
  operand (a b < q 2^64 for b < q).
* LZ inverse tail (gs_bfly_nr / gs_bfly_last_nr): stages 2, 1, 0 skip the sum reduction.
* Harvey [0, 4q) kernels for q < 2^62.
* csub's sign test: x - m in (-m, m) for x < 2m, m < 2^63.
"""
import pytest

import oracle as O

W = 1 << 64


def lz_schedule(n_stages):
    """(bounds before each stage, stages with the 8q reduction), mirroring lz_bound_before."""
    b, bounds, red = 1, [], []
    for s in range(n_stages):
        bounds.append(b)
        if b > 14:
            red.append(s)
            b = 8
        b += 2
    return bounds, red, b


def test_lz_schedule_matches_kernel_constants():
    bounds, red, out = lz_schedule(16)
    assert red == [7, 11, 15]                  # static_assert in modarith.cuh
    assert bounds[7] == 15 and out == 10
    _, red10, out10 = lz_schedule(10)
    assert red10 == [7] and out10 == 14        # N = 2^10: one reduced stage, output < 14q


@pytest.mark.parametrize("logn", list(range(4, 17)))
def test_lz_ct_ranges_fit_a_word(logn):
    q = (1 << 60) - 1                          # worst case of the lazy60 flag (every q < 2^60)
    bounds, red, out = lz_schedule(logn)
    for s, b in enumerate(bounds):
        x_max = b * q - 1                       # X input of stage s
        v_max = 2 * q - 1                       # Shoup product, [0, 2q)
        x_in = (8 * q - 1) if s in red else x_max
        if s in red:
            assert x_max < 16 * q and x_max - 8 * q < 8 * q   # csub(X, 8q) precondition
        assert x_in + v_max < W and x_in + 2 * q < W          # X' and Y' = x + 2q - v
    a_max = out * q - 1
    assert a_max * (q - 1) < q * W             # Montgomery operand (mont_mul, (0, 2q) result)
    assert out <= 16                            # canon16 handles [0, 16q)


def test_lz_inverse_tail_ranges():
    q = (1 << 60) - 1
    # stage 2: X, Y < 2q; stage 1: both < 4q; stage 0: both < 8q
    for by in (2, 4, 8):
        x_max = by * q - 1
        assert x_max + x_max < W                # X + Y
        assert x_max + by * q < W               # d = X + BY q - Y  (> 0 since Y < BY q)


def test_harvey_ranges_for_62_bit_moduli():
    q = (1 << 62) - 1
    assert 4 * q - 1 < W and 2 * q < 1 << 63   # [0, 4q) words, csub(X, 2q) sign test
    assert (4 * q - 1) * (q - 1) < q * W       # Montgomery of a [0, 4q) forward output


def test_csub_sign_test():
    for m in (3, 17, (1 << 61) - 1, (1 << 63) - 1):
        for x in (0, 1, m - 1, m, m + 1, 2 * m - 1):
            d = (x - m) % W
            signed = d - W if d >= 1 << 63 else d
            got = x if signed < 0 else d
            assert got == (x - m if x >= m else x)


def test_reading_c2_primes_take_the_lz_kernels():
    for logn, count in ((10, 1), (16, 60)):
        assert all(q < 1 << 60 for q in O.primes(logn, count))
