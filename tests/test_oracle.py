"""Pins for the CPU oracle (oracle/), independent of the oracle itself.

Each test checks the oracle against something other than its own code:
SPEC worked examples (tests/golden/spec_examples.json), the survey's
independently computed constants (tests/golden/survey_appendix_a.json),
closed forms, brute force on tiny inputs, Python big-integer evaluation of
the plain definitions, sieve / Lucas-certificate primality, and invariants
(round trip, linearity, negacyclic shift, convolution theorem).

P:n = PAPER.md line n, S:n = SPEC.md line n.
"""
import json
import math
import os
import random

import numpy as np
import pytest

import inputs
import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SPEC = json.load(open(os.path.join(GOLD, "spec_examples.json")))
APPA = json.load(open(os.path.join(GOLD, "survey_appendix_a.json")))


def brv_py(i, logn):
    return int(format(i, f"0{logn}b")[::-1], 2) if logn else 0


def eval_poly_py(a, x, q):
    """Horner evaluation of sum a_i x^i mod q with Python big ints."""
    acc = 0
    for c in reversed([int(v) for v in a]):
        acc = (acc * x + c) % q
    return acc


def ntt_definition_py(a, q, psi):
    """slot k = a(psi^{2 brv(k) + 1}) (Python big ints)."""
    n = len(a)
    logn = n.bit_length() - 1
    return [eval_poly_py(a, pow(psi, 2 * brv_py(k, logn) + 1, q), q) for k in range(n)]


def schoolbook_py(a, b, q):
    """a(x) b(x) mod (x^N + 1) by expanding the product, then x^N = -1."""
    n = len(a)
    full = [0] * (2 * n)
    for i in range(n):
        for j in range(n):
            full[i + j] += int(a[i]) * int(b[j])
    return [(full[k] - full[k + n]) % q for k in range(n)]


# --------------------------------------------------------------- scalars
def test_mulmod_spec_example():
    ex = SPEC["mod_mul"][0]
    assert O.mulmod(ex["a"], ex["b"], ex["q"]) == ex["out"]


def test_mulmod_powmod_against_python_bigints():
    rng = random.Random(1)
    for _ in range(2000):
        q = rng.randrange(2, 1 << 62)
        a, b = rng.randrange(q), rng.randrange(q)
        assert O.mulmod(a, b, q) == (a * b) % q
        e = rng.randrange(1 << 64)
        assert O.powmod(a, e, q) == pow(a, e, q)


def test_is_prime_matches_sieve():
    n = 1 << 16
    sieve = np.ones(n, dtype=bool)
    sieve[:2] = False
    for p in range(2, int(n ** 0.5) + 1):
        if sieve[p]:
            sieve[p * p :: p] = False
    for v in range(n):
        assert O.is_prime(v) == bool(sieve[v]), v


@pytest.mark.parametrize("n", [2047, 1373653, 25326001, 3215031751, 2152302898747,
                               3474749660383, 341550071728321, 3825123056546413051,
                               561, 1105, 1729, 2465, 2821, 6601])
def test_is_prime_rejects_strong_pseudoprimes_and_carmichaels(n):
    # Strong pseudoprimes to the first prime bases and Carmichael numbers.
    assert not O.is_prime(n)


def _pollard_rho(n):
    if n % 2 == 0:
        return 2
    rng = random.Random(n)
    while True:
        x = y = rng.randrange(2, n)
        c = rng.randrange(1, n)
        d = 1
        while d == 1:
            x = (x * x + c) % n
            y = (y * y + c) % n
            y = (y * y + c) % n
            d = math.gcd(abs(x - y), n)
        if d != n:
            return d


def _factor(n, out):
    if n == 1:
        return
    for p in range(2, 1000):
        while n % p == 0:
            out.add(p)
            n //= p
    if n == 1:
        return
    if n < 1000 * 1000:  # no factor below 1000 => prime
        out.add(n)
        return
    # Fermat test only used to decide when to stop splitting; the Lucas test
    # below re-proves the primality of the prime being certified.
    if all(pow(a, n - 1, n) == 1 for a in (2, 3, 5, 7, 11, 13, 17)):
        out.add(n)
        return
    d = _pollard_rho(n)
    _factor(d, out)
    _factor(n // d, out)


def lucas_certify(q):
    """Lucas primality proof: some a has a^{q-1}=1 and a^{(q-1)/p} != 1 for all p | q-1."""
    fs = set()
    _factor(q - 1, fs)
    for p in fs:  # factors must really divide and multiply back
        assert (q - 1) % p == 0
    for a in range(2, 200):
        if pow(a, q - 1, q) != 1:
            return False
        if all(pow(a, (q - 1) // p, q) != 1 for p in fs):
            return True
    return False


def test_q10_closed_form_and_certified():
    q = APPA["q10"]
    assert q == (1 << 60) - (1 << 14) + 1
    assert lucas_certify(q)
    assert O.primes(10, 4) == [q] + APPA["q10_next3"]


def test_primes_n65536_largest_first_and_certified():
    # Reading C2: the L largest primes < 2^60 with q = 1 mod 2N, descending.
    ps = O.primes(16, 60)
    g = APPA["p16"]
    assert ps[0] == (1 << 60) - (1 << 18) + 1 == g["p0"]
    assert [ps[1], ps[2], ps[3], ps[44], ps[59]] == [g["p1"], g["p2"], g["p3"], g["p44"], g["p59"]]
    assert sum(ps[:45]) % (1 << 64) == g["sum45_mod2_64"]
    assert sum(ps) % (1 << 64) == g["sum60_mod2_64"]
    two_n = 1 << 17
    for q in ps:
        assert q % two_n == 1 and q < (1 << 60) and q > (1 << 59)
        assert lucas_certify(q)
    # every skipped candidate k*2N+1 between them is composite (Fermat witness)
    for hi, lo in zip(ps[:10], ps[1:11]):
        for cand in range(hi - two_n, lo, -two_n):
            assert any(pow(a, cand - 1, cand) != 1 for a in (2, 3, 5, 7)), cand
    # nothing larger below 2^60 is a valid prime of that form
    for cand in range(ps[0] + two_n, 1 << 60, two_n):
        assert any(pow(a, cand - 1, cand) != 1 for a in (2, 3, 5, 7))


# ----------------------------------------------------------------- roots
@pytest.mark.parametrize("logn,q,psi", [tuple(x) for x in APPA["tiny"]["min_psi"]] + [(2, 17, 2)])
def test_min_psi_tiny_by_enumeration(logn, q, psi):
    n = 1 << logn
    assert O.min_psi(q, logn) == psi
    # brute force: smallest x with order exactly 2N
    def order(x):
        k, y = 1, x
        while y != 1:
            y = y * x % q
            k += 1
        return k
    smallest = min(x for x in range(2, q) if order(x) == 2 * n)
    assert smallest == psi


@pytest.mark.parametrize("q,logn,psi", [
    (APPA["q10"], 10, APPA["psi_q10_n1024"]),
    (APPA["p16"]["p0"], 16, APPA["p16"]["psi_p0"]),
    (APPA["p16"]["p44"], 16, APPA["p16"]["psi_p44"]),
])
def test_min_psi_large(q, logn, psi):
    n = 1 << logn
    got = O.min_psi(q, logn)
    assert got == psi
    assert pow(psi, n, q) == q - 1  # primitive 2N-th root (N power of two)
    assert O.is_primitive_2n_root(psi, q, logn)
    # minimality: enumerate all N primitive roots psi^{2t+1} with Python ints
    r2 = psi * psi % q
    cur, best = psi, psi
    for _ in range(n):
        best = min(best, cur)
        cur = cur * r2 % q
    assert best == psi


def test_is_primitive_root_rejects():
    q = 97
    assert not O.is_primitive_2n_root(1, q, 3)
    assert not O.is_primitive_2n_root(0, q, 3)
    assert not O.is_primitive_2n_root(q - 1, q, 3)  # order 2
    assert O.is_primitive_2n_root(8, q, 3)


def test_tables_are_powers():
    q, logn = 193, 5
    psi = O.min_psi(q, logn)
    fwd, inv, ninv = O.tables(q, psi, logn)
    psi_inv = pow(psi, -1, q)
    for i in range(1 << logn):
        assert fwd[i] == pow(psi, brv_py(i, logn), q)
        assert inv[i] == pow(psi_inv, brv_py(i, logn), q)
    assert ninv * (1 << logn) % q == 1
    t = APPA["tiny"]["n4_q17"]
    f4, _, _ = O.tables(17, t["psi"], 2)
    assert list(map(int, f4)) == t["fwd_table"]


# ------------------------------------------------------------- transforms
def test_ntt_worked_examples_n4_q17():
    t = APPA["tiny"]["n4_q17"]
    for a, want in t["ntt"]:
        assert list(map(int, O.ntt_fwd(a, 17, t["psi"]))) == want
    assert list(map(int, O.ntt_inv([1, 1, 1, 1], 17, t["psi"]))) == t["intt_ones"]


def test_ntt_worked_example_n16_q97():
    assert list(map(int, O.ntt_fwd(list(range(16)), 97, 19))) == APPA["tiny"]["n16_q97_ntt_0_to_15"]


def test_ntt_brute_force_all_inputs_n4_q17():
    """Every one of the 17^4 inputs at N=4, q=17 against the definition."""
    q, psi = 17, 2
    roots = [pow(psi, 2 * brv_py(k, 2) + 1, q) for k in range(4)]
    V = np.array([[pow(r, i, q) for i in range(4)] for r in roots], dtype=np.int64)
    grid = np.array(np.meshgrid(*[np.arange(q)] * 4, indexing="ij")).reshape(4, -1).T
    want = (grid @ V.T) % q
    data = grid.astype(np.uint64).reshape(-1, 1, 4)
    got = O.batch(O.OP_FWD, data, [q], [psi]).reshape(-1, 4)
    assert np.array_equal(got.astype(np.int64), want)
    back = O.batch(O.OP_INV, got.reshape(-1, 1, 4), [q], [psi]).reshape(-1, 4)
    assert np.array_equal(back, grid.astype(np.uint64))


@pytest.mark.parametrize("logn,q", [(3, 17), (3, 97), (4, 97), (4, 193), (5, 193), (6, 257),
                                    (5, 1152921504606830593), (6, 1152921504606584833)])
def test_ntt_matches_python_definition(logn, q):
    n = 1 << logn
    psi = O.min_psi(q, logn)
    rng = np.random.default_rng(logn * 1000 + q % 1000)
    vecs = [np.eye(n, dtype=np.uint64)[j] for j in range(n)]
    vecs += [np.array([rng.integers(0, q) for _ in range(n)], dtype=np.uint64) for _ in range(20)]
    for a in vecs:
        want = ntt_definition_py(a, q, psi)
        assert list(map(int, O.ntt_fwd(a, q, psi))) == want
        assert list(map(int, O.naive_ntt(a, q, psi))) == want
        assert list(map(int, O.ntt_inv(np.array(want, dtype=np.uint64), q, psi))) == list(map(int, a))


def test_ntt_delta_and_ones():
    # S:162 NTT(delta_0) = 1...1 ; S:169 INTT(1...1) = delta_0
    for logn, q in [(4, 97), (10, APPA["q10"]), (16, APPA["p16"]["p0"])]:
        n = 1 << logn
        psi = O.min_psi(q, logn)
        d = np.zeros(n, dtype=np.uint64)
        d[0] = 1
        assert np.all(O.ntt_fwd(d, q, psi) == 1)
        back = O.ntt_inv(np.ones(n, dtype=np.uint64), q, psi)
        assert back[0] == 1 and np.all(back[1:] == 0)


def test_ntt_monomials_closed_form():
    """NTT(x^j)[k] = psi^{(2 brv(k) + 1) j}: pins values and the bo order."""
    q = APPA["q10"]
    logn = 10
    n = 1 << logn
    psi = APPA["psi_q10_n1024"]
    for j in [0, 1, 2, 3, 511, 512, 1023]:
        a = np.zeros(n, dtype=np.uint64)
        a[j] = 1
        got = O.ntt_fwd(a, q, psi)
        for k in range(0, n, 37):
            assert int(got[k]) == pow(psi, (2 * brv_py(k, logn) + 1) * j, q)


def test_negacyclic_shift_invariant_n65536():
    """NTT(x a mod x^N+1)[k] = psi^{2 brv(k)+1} NTT(a)[k]; O(N) check at 2^16."""
    q = APPA["p16"]["p44"]
    logn = 16
    psi = APPA["p16"]["psi_p44"]
    a = inputs.residues(7, 1, [q], 1 << logn)[0, 0]
    xa = np.roll(a, 1)
    xa[0] = (q - int(a[-1])) % q
    A = O.ntt_fwd(a, q, psi)
    XA = O.ntt_fwd(xa, q, psi)
    ks = np.random.default_rng(3).integers(0, 1 << logn, 200)
    for k in ks:
        k = int(k)
        z = pow(psi, 2 * brv_py(k, logn) + 1, q)
        assert int(XA[k]) == z * int(A[k]) % q


def test_linearity():
    q = APPA["q10"]
    psi = APPA["psi_q10_n1024"]
    a = inputs.residues(1, 1, [q], 1024)[0, 0]
    b = inputs.residues(2, 1, [q], 1024)[0, 0]
    al, be = 123456789, 987654321987
    comb = np.array([(al * int(x) + be * int(y)) % q for x, y in zip(a, b)], dtype=np.uint64)
    A, B, C = O.ntt_fwd(a, q, psi), O.ntt_fwd(b, q, psi), O.ntt_fwd(comb, q, psi)
    assert all(int(C[k]) == (al * int(A[k]) + be * int(B[k])) % q for k in range(1024))


def test_roundtrip_many_sizes():
    # S:164 round trip, here 20 trials per N (the GPU tests run more).
    rng = np.random.default_rng(5)
    for logn in [1, 2, 3, 4, 10, 12, 13, 16]:
        n = 1 << logn
        q = O.primes(logn, 1)[0]
        psi = O.min_psi(q, logn)
        trials = 20 if logn <= 12 else 2
        for t in range(trials):
            a = inputs.residues(int(rng.integers(1 << 30)), 1, [q], n)[0, 0]
            assert np.array_equal(O.ntt_inv(O.ntt_fwd(a, q, psi), q, psi), a)


def test_naive_intt_at_inverts_definition():
    q, logn = 257, 6
    psi = O.min_psi(q, logn)
    a = np.arange(64, dtype=np.uint64) * 3 % q
    A = O.ntt_fwd(a, q, psi)
    for i in range(64):
        assert O.naive_intt_at(A, q, psi, i) == int(a[i])


# -------------------------------------------------------------- products
def test_schoolbook_spec_examples():
    for ex in SPEC["schoolbook"]:
        assert list(map(int, O.schoolbook(ex["a"], ex["b"], ex["q"]))) == ex["out"]


def test_schoolbook_matches_python_expansion():
    rng = random.Random(9)
    for logn, q in [(2, 17), (3, 97), (5, 193), (6, 1152921504606830593)]:
        n = 1 << logn
        for _ in range(10):
            a = [rng.randrange(q) for _ in range(n)]
            b = [rng.randrange(q) for _ in range(n)]
            want = schoolbook_py(a, b, q)
            assert list(map(int, O.schoolbook(a, b, q))) == want
            assert O.schoolbook_at(a, b, q, n - 1) == want[n - 1]


def test_convolution_theorem_spec():
    # N=16, q=97, 50 random pairs: INTT(NTT(a).NTT(b)) = schoolbook
    ex = SPEC["convolution_theorem"]
    q, n = ex["q"], ex["n"]
    psi = O.min_psi(q, 4)
    rng = random.Random(11)
    for _ in range(ex["pairs"]):
        a = [rng.randrange(q) for _ in range(n)]
        b = [rng.randrange(q) for _ in range(n)]
        c = O.ntt_inv(O.pointwise(O.ntt_fwd(a, q, psi), O.ntt_fwd(b, q, psi), q), q, psi)
        assert list(map(int, c)) == schoolbook_py(a, b, q)


@pytest.mark.parametrize("logn", [3, 4, 6, 10])
def test_polymul_batch_matches_schoolbook(logn):
    # SPEC acceptance #2: N in {8, 16, 64, 1024}
    n = 1 << logn
    ps = O.primes(logn, 2)
    psi = [O.min_psi(q, logn) for q in ps]
    B = 3 if logn == 10 else 8
    a = inputs.residues(21, B, ps, n)
    b = inputs.residues(22, B, ps, n)
    c = O.batch(O.OP_POLYMUL, a, ps, psi, b=b, n_threads=2)
    for bi in range(B):
        for l, q in enumerate(ps):
            if logn <= 6:
                assert list(map(int, c[bi, l])) == schoolbook_py(a[bi, l], b[bi, l], q)
            else:
                for k in (0, 1, n // 2, n - 1):
                    assert int(c[bi, l, k]) == O.schoolbook_at(a[bi, l], b[bi, l], q, k)
    # eval-form operand and broadcast give the same result
    bhat = O.batch(O.OP_FWD, b, ps, psi)
    c2 = O.batch(O.OP_POLYMUL_EVAL, a, ps, psi, b=bhat)
    assert np.array_equal(c, c2)
    c3 = O.batch(O.OP_POLYMUL_EVAL, a, ps, psi, b=bhat[:1], b_broadcast=True)
    for bi in range(B):
        assert np.array_equal(c3[bi], O.batch(O.OP_POLYMUL_EVAL, a[bi:bi + 1], ps, psi, b=bhat[:1])[0])


def test_batch_threads_deterministic():
    ps = O.primes(10, 3)
    psi = [O.min_psi(q, 10) for q in ps]
    a = inputs.residues(3, 5, ps, 1024)
    r1 = O.batch(O.OP_FWD, a, ps, psi, n_threads=1)
    r8 = O.batch(O.OP_FWD, a, ps, psi, n_threads=8)
    assert np.array_equal(r1, r8)
    for bi in range(5):
        for l in range(3):
            assert np.array_equal(r1[bi, l], O.ntt_fwd(a[bi, l], ps[l], psi[l]))


def test_oracle_rejects_noncanonical():
    with pytest.raises(ValueError):
        O.ntt_fwd([17, 0, 0, 0], 17, 2)


# ----------------------------------------------------- seeded config digests
def test_generator_known_answers():
    z = inputs.splitmix64(0, np.arange(3))
    assert [int(v) for v in z] == [int(s, 16) for s in APPA["splitmix64_seed0"]]


def test_cfg1_seeded_values():
    g = APPA["cfg1_seed0"]
    q = APPA["q10"]
    psi = APPA["psi_q10_n1024"]
    a = inputs.residues(0, 1, [q], 1024)
    b = inputs.residues(1, 1, [q], 1024)
    assert list(map(int, a[0, 0, :4])) == g["a_head"]
    A = O.batch(O.OP_FWD, a, [q], [psi])[0, 0]
    assert list(map(int, A[:4])) == g["ntt_head"] and int(A[-1]) == g["ntt_last"]
    assert inputs.digest(A) == (g["ntt_sum"], g["ntt_wsum"])
    c = O.batch(O.OP_POLYMUL, a, [q], [psi], b=b)[0, 0]
    assert list(map(int, c[:4])) == g["polymul_head"]
    assert inputs.digest(c) == (g["polymul_sum"], g["polymul_wsum"])
    for k in (0, 1, 2, 3, 700, 1023):
        assert int(c[k]) == O.schoolbook_at(a[0, 0], b[0, 0], q, k)


@pytest.mark.slow
def test_cfg3_seeded_digests():
    g = APPA["cfg3_seed0"]
    ps = O.primes(16, 45)
    sel = [0, 44]
    mods = [ps[i] for i in sel]
    psi = [O.min_psi(q, 16) for q in mods]
    a = inputs.residues_limbs(0, 1, mods[:1], 1 << 16, 0, 45)
    a = np.concatenate([a, inputs.residues_limbs(0, 1, mods[1:], 1 << 16, 44, 45)], axis=1)
    b = np.concatenate([inputs.residues_limbs(1, 1, mods[:1], 1 << 16, 0, 45),
                        inputs.residues_limbs(1, 1, mods[1:], 1 << 16, 44, 45)], axis=1)
    A = O.batch(O.OP_FWD, a, mods, psi, n_threads=2)
    C = O.batch(O.OP_POLYMUL, a, mods, psi, b=b, n_threads=2)
    for li, key in enumerate(["limb0", "limb44"]):
        assert int(a[0, li, 0]) == g[key]["a0"]
        assert inputs.digest(A[0, li]) == (g[key]["ntt_sum"], g[key]["ntt_wsum"])
        assert inputs.digest(C[0, li]) == (g[key]["polymul_sum"], g[key]["polymul_wsum"])
    # sampled schoolbook at full size
    for k in (0, 12345, 65535):
        assert int(C[0, 0, k]) == O.schoolbook_at(a[0, 0], b[0, 0], mods[0], k)


# ------------------------------------------------------------- automorph (f4)
def test_automorph_monomials_closed_form():
    """sigma_g(x^j) = x^{jg mod 2N}, with x^N = -1 (P:248 Automorph, P:194 ring)."""
    q, logn = 97, 4
    n = 1 << logn
    for g in (1, 3, 5, 7, 31):
        for j in range(n):
            a = np.zeros(n, dtype=np.uint64)
            a[j] = 1
            out = O.automorph(a, q, g)
            t = j * g % (2 * n)
            want = np.zeros(n, dtype=np.uint64)
            want[t % n] = 1 if t < n else q - 1
            assert np.array_equal(out, want)


def test_automorph_is_ring_homomorphism_and_composes():
    q = 1152921504606830593
    n = 64
    rng = random.Random(3)
    a = [rng.randrange(q) for _ in range(n)]
    b = [rng.randrange(q) for _ in range(n)]
    for g in (3, 5, 127):
        lhs = O.automorph(schoolbook_py(a, b, q), q, g)
        rhs = schoolbook_py(list(map(int, O.automorph(a, q, g))), list(map(int, O.automorph(b, q, g))), q)
        assert list(map(int, lhs)) == rhs
    for g, h in ((3, 5), (7, 9), (127, 3)):
        assert np.array_equal(O.automorph(O.automorph(a, q, h), q, g), O.automorph(a, q, g * h % (2 * n)))
    assert np.array_equal(O.automorph(a, q, 1), np.array(a, dtype=np.uint64))


def test_automorph_ntt_domain_is_slot_permutation():
    """NTT(sigma_g(a))[k] = NTT(a)[pi(k)], 2 brv(pi(k)) + 1 = (2 brv(k) + 1) g mod 2N."""
    logn = 6
    n = 1 << logn
    q = O.primes(logn, 1)[0]
    psi = O.min_psi(q, logn)
    a = inputs.residues(5, 1, [q], n)[0, 0]
    A = O.ntt_fwd(a, q, psi)
    for g in (3, 5, 2 * n - 1):
        S = O.ntt_fwd(O.automorph(a, q, g), q, psi)
        for k in range(n):
            e = (2 * brv_py(k, logn) + 1) * g % (2 * n)
            assert int(S[k]) == int(A[brv_py((e - 1) // 2, logn)])


# ------------------------------------------------ TFHE external product (f1)
def test_decompose_spec_example():
    # B_g=4, l=2, q=16, constant 7 -> digits (-1, 2): -1*1 + 2*4 = 7
    d = O.decompose(7, 16, 2, 2)
    assert d == [16 - 1, 2]


def test_decompose_recomposes_exactly_and_digits_bounded():
    rng = random.Random(17)
    q = 1152921504606830593
    for bg, l in ((20, 3), (15, 4), (10, 6), (30, 2)):
        B = 1 << bg
        assert B ** l >= q
        vals = [0, 1, q - 1, (q - 1) // 2, (q + 1) // 2] + [rng.randrange(q) for _ in range(500)]
        for v in vals:
            ds = O.decompose(v, q, bg, l)
            signed = [d if d <= q // 2 else d - q for d in ds]
            assert all(-B // 2 <= s < B // 2 for s in signed[:-1])
            assert -B // 2 <= signed[-1] <= B // 2
            assert sum(s * B ** j for j, s in enumerate(signed)) % q == v


def _gadget_rgsw_hat(q, psi, n, bg, l):
    """Trivial RGSW of 1 with zero noise: row (t, j) = B^j e_t (gadget matrix G), NTT form."""
    z = np.zeros((2 * l, 2, n), dtype=np.uint64)
    for t in range(2):
        for j in range(l):
            row = np.zeros(n, dtype=np.uint64)
            row[0] = pow(2, bg * j, q)
            z[t * l + j, t] = O.ntt_fwd(row, q, psi)
    return z


def test_external_product_with_gadget_matrix_is_identity():
    """Decompose-then-recompose is exact, so c boxtimes G = c."""
    for logn, bg, l in ((4, 20, 3), (10, 20, 3), (10, 30, 2)):
        n = 1 << logn
        q = O.primes(logn, 1)[0]
        psi = O.min_psi(q, logn)
        c = inputs.residues(9, 2, [q], n)[:, 0, :]
        out = O.external_product(c, _gadget_rgsw_hat(q, psi, n, bg, l), q, psi, bg, l)
        assert np.array_equal(out, c)


def test_external_product_matches_schoolbook_expansion():
    logn, bg, l = 4, 20, 3
    n = 1 << logn
    q = O.primes(logn, 1)[0]
    psi = O.min_psi(q, logn)
    rng = np.random.default_rng(4)
    c = inputs.residues(11, 2, [q], n)[:, 0, :]
    z = inputs.residues(12, 2 * l * 2, [q], n).reshape(2 * l, 2, n)
    zhat = np.stack([np.stack([O.ntt_fwd(z[r, i], q, psi) for i in range(2)]) for r in range(2 * l)])
    out = O.external_product(c, zhat, q, psi, bg, l)
    for i in range(2):
        acc = [0] * n
        for t in range(2):
            digs = [O.decompose(int(v), q, bg, l) for v in c[t]]
            for j in range(l):
                D = [digs[k][j] for k in range(n)]
                prod = schoolbook_py(D, list(map(int, z[t * l + j, i])), q)
                acc = [(x + y) % q for x, y in zip(acc, prod)]
        assert list(map(int, out[i])) == acc


# ---------------------------------------------------------------- BConv (f2)
def _crt(residues, mods):
    M = 1
    for m in mods:
        M *= m
    x = 0
    for r, m in zip(residues, mods):
        Mi = M // m
        x += int(r) * Mi * pow(Mi, -1, m)
    return x % M, M


def test_bconv_is_x_plus_alpha_q_with_alpha_below_L():
    """BConv = X + alpha Q (0 <= alpha < L) with X the exact CRT value (big ints)."""
    qs = O.primes(10, 5)
    ps = O.primes(11, 4)   # disjoint basis (q = 1 mod 2^12)
    rng = random.Random(5)
    n = 16
    x = np.array([[rng.randrange(q) for _ in range(n)] for q in qs], dtype=np.uint64)
    x[:, 0] = 0
    x[:, 1] = [q - 1 for q in qs]
    out = O.bconv(x, qs, ps)
    Q = 1
    for q in qs:
        Q *= q
    for c in range(n):
        X, _ = _crt(x[:, c], qs)
        ys = [int(x[i, c]) * pow(Q // qs[i], -1, qs[i]) % qs[i] for i in range(len(qs))]
        S = sum(y * (Q // q) for y, q in zip(ys, qs))
        alpha = (S - X) // Q
        assert (S - X) % Q == 0 and 0 <= alpha < len(qs)
        for j, p in enumerate(ps):
            assert int(out[j, c]) == (X + alpha * Q) % p


def test_bconv_zero_and_single_limb():
    """x = 0 maps to 0; with L = 1 (Q = q_0, alpha = 0) BConv is x mod p_j exactly."""
    qs = O.primes(10, 3)
    ps = O.primes(11, 2)
    x = np.zeros((3, 4), dtype=np.uint64)
    assert not O.bconv(x, qs, ps).any()
    x1 = np.array([[5, qs[0] - 1, 123456789, 0]], dtype=np.uint64)
    out = O.bconv(x1, qs[:1], ps)
    for j, p in enumerate(ps):
        assert list(map(int, out[j])) == [int(v) % p for v in x1[0]]
