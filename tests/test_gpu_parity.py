"""GPU parity: the sm_100a kernels through the C ABI versus the CPU oracle,
bit-exact on every element (integer work, BASELINE.json north_star).

Inputs come from inputs/ (SplitMix64 + Lemire, seeded); expected values come
only from oracle/.  P:n = PAPER.md line n.
"""
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

ALL_LOGN = list(range(4, 17))


def _plan(logn, limbs):
    ps, psi = params(logn, limbs)
    p = R.Plan(logn, ps)
    assert p.psi() == list(psi)  # plan's reading-C1 psi equals the oracle's
    return p, ps, psi


def _batch_for(logn):
    return {4: 37, 5: 33, 6: 19, 7: 9, 8: 9, 9: 5, 10: 7}.get(logn, 2)


@pytest.mark.parametrize("logn", ALL_LOGN)
def test_forward_inverse_all_sizes(logn):
    limbs = 3
    B = _batch_for(logn)
    p, ps, psi = _plan(logn, limbs)
    n = 1 << logn
    a = inputs.residues(100 + logn, B, ps, n)
    want = O.batch(O.OP_FWD, a, ps, psi, n_threads=8)
    da = to_dev(a)
    dout = empty_dev(a.shape)
    R.ntt_forward(p, dout, da)
    got = from_dev(dout)
    assert np.array_equal(got, want)
    # inverse of the oracle's forward output must give back a
    dback = empty_dev(a.shape)
    R.ntt_inverse(p, dback, to_dev(want))
    assert np.array_equal(from_dev(dback), a)
    # inverse on random eval-domain input vs the oracle inverse
    A = inputs.residues(200 + logn, B, ps, n)
    R.ntt_inverse(p, dback, to_dev(A))
    assert np.array_equal(from_dev(dback), O.batch(O.OP_INV, A, ps, psi, n_threads=8))


@pytest.mark.parametrize("logn", ALL_LOGN)
@pytest.mark.parametrize("bcast", [False, True])
def test_polymul_all_sizes(logn, bcast):
    limbs = 2
    B = _batch_for(logn)
    p, ps, psi = _plan(logn, limbs)
    n = 1 << logn
    a = inputs.residues(300 + logn, B, ps, n)
    b = inputs.residues(400 + logn, 1 if bcast else B, ps, n)
    want = O.batch(O.OP_POLYMUL, a, ps, psi, b=b, b_broadcast=bcast, n_threads=8)
    bhat = O.batch(O.OP_FWD, b, ps, psi, n_threads=8)
    dc = empty_dev(a.shape)
    R.polymul(p, dc, to_dev(a), to_dev(b), b_is_eval=False, b_broadcast=bcast)
    assert np.array_equal(from_dev(dc), want)
    R.polymul(p, dc, to_dev(a), to_dev(bhat), b_is_eval=True, b_broadcast=bcast)
    assert np.array_equal(from_dev(dc), want)
    # sampled schoolbook on the GPU result itself
    got = from_dev(dc)
    for k in (0, n // 3, n - 1):
        assert int(got[0, 0, k]) == O.schoolbook_at(a[0, 0], b[0, 0], ps[0], k)


@pytest.mark.parametrize("logn", [4, 10, 12, 16])
def test_pointwise(logn):
    p, ps, psi = _plan(logn, 3)
    n = 1 << logn
    B = 3
    a = inputs.residues(5, B, ps, n)
    b = inputs.residues(6, B, ps, n)
    dc = empty_dev(a.shape)
    R.pointwise_mul(p, dc, to_dev(a), to_dev(b))
    want = np.stack([np.stack([O.pointwise(a[i, l], b[i, l], ps[l]) for l in range(3)]) for i in range(B)])
    assert np.array_equal(from_dev(dc), want)
    R.pointwise_mul(p, dc, to_dev(a), to_dev(b[:1]), b_broadcast=True)
    want = np.stack([np.stack([O.pointwise(a[i, l], b[0, l], ps[l]) for l in range(3)]) for i in range(B)])
    assert np.array_equal(from_dev(dc), want)


@pytest.mark.parametrize("logn", [4, 7, 10, 11, 16])
def test_edge_inputs(logn):
    """zeros, all q-1 (max lazy range), delta_0, delta_{N-1}, alternating, monomials."""
    n = 1 << logn
    p, ps, psi = _plan(logn, 2)
    rows = []
    for l, q in enumerate(ps):
        pass
    vecs = []
    z = np.zeros((2, n), dtype=np.uint64)
    vecs.append(z.copy())
    vecs.append(np.array([[q - 1] * n for q in ps], dtype=np.uint64))
    d0 = z.copy(); d0[:, 0] = 1; vecs.append(d0)
    dl = z.copy(); dl[:, -1] = 1; vecs.append(dl)
    alt = np.array([[0 if i % 2 == 0 else q - 1 for i in range(n)] for q in ps], dtype=np.uint64)
    vecs.append(alt)
    for j in (1, n // 2, n - 2):
        m = z.copy(); m[:, j] = 1; vecs.append(m)
    a = np.stack(vecs)  # [B][L][N]
    want = O.batch(O.OP_FWD, a, ps, psi)
    d = empty_dev(a.shape)
    R.ntt_forward(p, d, to_dev(a))
    got = from_dev(d)
    assert np.array_equal(got, want)
    assert np.all(got[2] == 1)  # NTT(delta_0) = 1
    R.ntt_inverse(p, d, to_dev(np.ones_like(a)))
    back = from_dev(d)
    assert np.all(back[:, :, 0] == 1) and np.all(back[:, :, 1:] == 0)
    # polymul of extremes: (q-1 ... ) * (q-1 ...)
    c = empty_dev(a.shape)
    R.polymul(p, c, to_dev(a), to_dev(a[::-1].copy()))
    assert np.array_equal(from_dev(c), O.batch(O.OP_POLYMUL, a, ps, psi, b=a[::-1].copy()))


@pytest.mark.parametrize("logn", [6, 10, 13, 16])
def test_in_place(logn):
    p, ps, psi = _plan(logn, 2)
    a = inputs.residues(8, 3, ps, 1 << logn)
    d = to_dev(a)
    R.ntt_forward(p, d, d)
    assert np.array_equal(from_dev(d), O.batch(O.OP_FWD, a, ps, psi))
    R.ntt_inverse(p, d, d)
    assert np.array_equal(from_dev(d), a)
    b = inputs.residues(9, 3, ps, 1 << logn)
    R.polymul(p, d, d, to_dev(b))
    assert np.array_equal(from_dev(d), O.batch(O.OP_POLYMUL, a, ps, psi, b=b))


def test_tiny_prime_spec_example():
    """q = 97, N = 16 on the GPU: NTT(0..15) worked value and S:171 convolution."""
    p = R.Plan(4, [97])
    assert p.psi() == [19]
    a = np.arange(16, dtype=np.uint64).reshape(1, 1, 16)
    d = empty_dev(a.shape)
    R.ntt_forward(p, d, to_dev(a))
    assert list(map(int, from_dev(d).ravel())) == [13, 72, 27, 49, 55, 96, 18, 8, 60, 8, 32, 51, 36, 67, 67, 20]
    rng = np.random.default_rng(0)
    A = rng.integers(0, 97, (50, 1, 16)).astype(np.uint64)
    Bm = rng.integers(0, 97, (50, 1, 16)).astype(np.uint64)
    R.polymul(p, empty_dev(A.shape), to_dev(A), to_dev(Bm))
    c = empty_dev(A.shape)
    R.polymul(p, c, to_dev(A), to_dev(Bm))
    got = from_dev(c)
    for i in range(50):
        assert np.array_equal(got[i, 0], O.schoolbook(A[i, 0], Bm[i, 0], 97))


def test_explicit_psi():
    logn = 10
    ps, _ = params(logn, 1)
    q = ps[0]
    psi_min = O.min_psi(q, logn)
    other = pow(psi_min, 3, q)  # also a primitive 2N-th root (odd power)
    p = R.Plan(logn, [q], psi=[other])
    a = inputs.residues(1, 2, [q], 1 << logn)
    d = empty_dev(a.shape)
    R.ntt_forward(p, d, to_dev(a))
    assert np.array_equal(from_dev(d), O.batch(O.OP_FWD, a, [q], [other]))


def test_roundtrip_100_trials():
    # SPEC S:164 / acceptance #1: 100 trials per N in {2^10, 2^12, 2^13, 2^16}
    for logn in (10, 12, 13, 16):
        p, ps, psi = _plan(logn, 1)
        a = inputs.residues(77, 100, ps, 1 << logn)
        d = to_dev(a)
        R.ntt_forward(p, d, d)
        R.ntt_inverse(p, d, d)
        assert np.array_equal(from_dev(d), a)


def test_cfg1_seeded_digest_matches_survey():
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "survey_appendix_a.json")))
    q = g["q10"]
    p = R.Plan(10, [q])
    a = inputs.residues(0, 1, [q], 1024)
    b = inputs.residues(1, 1, [q], 1024)
    d = empty_dev(a.shape)
    R.ntt_forward(p, d, to_dev(a))
    assert inputs.digest(from_dev(d)) == (g["cfg1_seed0"]["ntt_sum"], g["cfg1_seed0"]["ntt_wsum"])
    R.polymul(p, d, to_dev(a), to_dev(b))
    assert inputs.digest(from_dev(d)) == (g["cfg1_seed0"]["polymul_sum"], g["cfg1_seed0"]["polymul_wsum"])


# ------------------------------------------------------------- full configs
def test_cfg2_full_bitexact():
    """TFHE batch: N=2^10, 4096 polys: NTT -> (.) b_hat -> INTT, every element."""
    ps, psi = params(10, 1)
    p = R.Plan(10, ps)
    a = inputs.residues(0, 4096, ps, 1024)
    b = inputs.residues(1, 4096, ps, 1024)
    bhat = O.batch(O.OP_FWD, b, ps, psi, n_threads=8)
    d = empty_dev(a.shape)
    R.ntt_forward(p, d, to_dev(a))
    assert np.array_equal(from_dev(d), O.batch(O.OP_FWD, a, ps, psi, n_threads=8))
    R.polymul(p, d, to_dev(a), to_dev(bhat), b_is_eval=True)
    assert np.array_equal(from_dev(d), O.batch(O.OP_POLYMUL_EVAL, a, ps, psi, b=bhat, n_threads=8))


def test_cfg3_full_bitexact():
    """CKKS HMUL-sized: N=2^16, 45 limbs, NTT -> (.) b_hat -> INTT (reading C8)."""
    ps, psi = params(16, 45)
    p = R.Plan(16, ps)
    a = inputs.residues(0, 1, ps, 1 << 16)
    b = inputs.residues(1, 1, ps, 1 << 16)
    bhat = O.batch(O.OP_FWD, b, ps, psi, n_threads=8)
    d = empty_dev(a.shape)
    R.polymul(p, d, to_dev(a), to_dev(bhat), b_is_eval=True)
    got = from_dev(d)
    assert np.array_equal(got, O.batch(O.OP_POLYMUL_EVAL, a, ps, psi, b=bhat, n_threads=8))
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "survey_appendix_a.json")))["cfg3_seed0"]
    assert inputs.digest(got[0, 0]) == (g["limb0"]["polymul_sum"], g["limb0"]["polymul_wsum"])
    assert inputs.digest(got[0, 44]) == (g["limb44"]["polymul_sum"], g["limb44"]["polymul_wsum"])


def test_cfg4_full_bitexact():
    """N=2^16, 60 limbs x 8 polys, forward + inverse, every element."""
    ps, psi = params(16, 60)
    p = R.Plan(16, ps)
    a = inputs.residues(0, 8, ps, 1 << 16)
    d = to_dev(a)
    R.ntt_forward(p, d, d)
    fwd = from_dev(d)
    assert np.array_equal(fwd, O.batch(O.OP_FWD, a, ps, psi, n_threads=8))
    R.ntt_inverse(p, d, d)
    assert np.array_equal(from_dev(d), a)


def test_streams_and_concurrency():
    ps, psi = params(16, 4)
    p = R.Plan(16, ps)
    a = inputs.residues(3, 2, ps, 1 << 16)
    want = O.batch(O.OP_FWD, a, ps, psi)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    d1, d2 = to_dev(a), to_dev(a)
    torch.cuda.synchronize()
    R.ntt_forward(p, d1, d1, stream=s1)
    R.ntt_forward(p, d2, d2, stream=s2)
    torch.cuda.synchronize()
    assert np.array_equal(from_dev(d1), want) and np.array_equal(from_dev(d2), want)


def test_execute_host_roundtrip():
    ps, psi = params(10, 1)
    p = R.Plan(10, ps)
    a = inputs.residues(4, 64, ps, 1024)
    hin = torch.from_numpy(a.view(np.int64).copy()).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    ws = empty_dev(a.shape)
    R.execute_host(p, R.OP_FORWARD, hout, hin, ws)
    torch.cuda.synchronize()
    assert np.array_equal(hout.numpy().view(np.uint64), O.batch(O.OP_FWD, a, ps, psi))


def test_batch_zero_is_noop_and_errors():
    ps, _ = params(10, 1)
    p = R.Plan(10, ps)
    d = empty_dev((1, 1, 1024))
    R.ntt_forward(p, d, d, batch=0)
    with pytest.raises(R.RntError) as e:
        R.ntt_forward(p, d.data_ptr() + 8, d, batch=1)  # misaligned raw pointer reaches the C ABI check
    assert e.value.code == R.RNT_E_INVALID_ARG


def test_binding_rejects_undersized_or_mistyped_buffers():
    """The Python binding checks element size, device and the words each call touches
    before the C ABI (which cannot see tensor sizes) runs."""
    ps, psi = params(10, 2)
    p = R.Plan(10, ps)
    a = empty_dev((3, 2, 1024))
    small = empty_dev((2, 2, 1024))
    with pytest.raises(ValueError):
        R.ntt_forward(p, small, a)                                   # out smaller than the batch
    with pytest.raises(ValueError):
        R.ntt_forward(p, a, torch.zeros((3, 2, 1024), dtype=torch.int32, device="cuda"))   # 4-byte elements
    with pytest.raises(ValueError):
        R.polymul(p, a, a.clone(), small[:1], b_is_eval=True)         # b of one polynomial without broadcast
    R.polymul(p, a, a.clone().zero_(), small[:1].zero_(), b_is_eval=True, b_broadcast=True)   # fine when broadcast
    with pytest.raises(ValueError):
        R.pointwise_mul(p, a, a.clone(), small)                       # b_hat of 2 polynomials for a batch of 3
    with pytest.raises(ValueError):
        R.automorph(p, small, a, 3)
    with pytest.raises(ValueError):
        R.ntt_forward(p, a, a.cpu())                                  # host tensor
    pe = R.Plan(10, ps[:1])
    c = empty_dev((4, 2, 1024))
    with pytest.raises(ValueError):
        R.external_product(pe, empty_dev((3, 2, 1024)), c, empty_dev((6, 2, 1024)), 20, 3)   # out too small
    with pytest.raises(ValueError):
        R.external_product(pe, c.clone(), c, empty_dev((5, 2, 1024)), 20, 3)                # rgsw rows missing
    qs = ps[:1]
    qp, qpp = R.Plan(10, qs), R.Plan(10, ps)
    ks = R.KeySwitch(qp, qpp, 1)
    with pytest.raises(ValueError):
        ks(empty_dev((1, 1, 1024)), empty_dev((1, 1024)), empty_dev((1, 2, 2, 1024)))      # out needs [2][L][N]
    with pytest.raises(ValueError):
        ks(empty_dev((2, 1, 1024)), empty_dev((1, 1024)), empty_dev((1, 2, 1, 1024)))      # evk needs [dnum][2][L+K][N]
    bc = R.BConv(qp, qpp)
    with pytest.raises(ValueError):
        bc(empty_dev((3, 1, 1024)), empty_dev((3, 1, 1024)))                               # out needs K = 2 limbs
    hin = torch.zeros((3, 2, 1024), dtype=torch.int64).pin_memory()
    with pytest.raises(ValueError):
        R.execute_host(p, R.OP_FORWARD, torch.zeros((2, 2, 1024), dtype=torch.int64), hin, a)   # host out too small


# Shapes above the 32 MiB chunk: (10,1,10000) 3 chunks over polynomials (4096, 4096, 1808),
# (10,2,5000) 3 (2048, 2048, 904), (16,70,1) 2 limb windows (64 + 6), (16,9,9) 2 (7 + 2).
@pytest.mark.parametrize("logn,limbs,batch,op", [(10, 1, 10000, "fwd"), (10, 2, 5000, "polymul_eval"),
                                                 (16, 70, 1, "polymul_eval"), (16, 9, 9, "inv"),
                                                 (16, 70, 1, "polymul"), (16, 45, 1, "polymul_eval")])
def test_execute_host_chunked_pipeline(logn, limbs, batch, op):
    """rnt_execute_host splits large jobs into 32 MiB chunks over 3 internal streams."""
    ps, psi = params(logn, limbs)
    p = R.Plan(logn, ps)
    a = inputs.residues(12, batch, ps, 1 << logn)
    hin = torch.from_numpy(a.view(np.int64).copy()).pin_memory()
    hout = torch.zeros_like(hin).pin_memory()
    ws = empty_dev(a.shape)
    if op == "fwd":
        R.execute_host(p, R.OP_FORWARD, hout, hin, ws)
        want = O.batch(O.OP_FWD, a, ps, psi, n_threads=8)
    elif op == "inv":
        R.execute_host(p, R.OP_INVERSE, hout, hin, ws)
        want = O.batch(O.OP_INV, a, ps, psi, n_threads=8)
    else:
        b = inputs.residues(13, batch, ps, 1 << logn)
        if op == "polymul_eval":
            bhat = O.batch(O.OP_FWD, b, ps, psi, n_threads=8)
            R.execute_host(p, R.OP_POLYMUL_EVAL, hout, hin, ws, b_dev=to_dev(bhat))
        else:
            R.execute_host(p, R.OP_POLYMUL, hout, hin, ws, b_dev=to_dev(b))
        want = O.batch(O.OP_POLYMUL, a, ps, psi, b=b, n_threads=8)
    torch.cuda.synchronize()
    assert np.array_equal(hout.numpy().view(np.uint64), want)


@pytest.mark.parametrize("logn,limbs", [(11, 4), (12, 5), (14, 7), (16, 45)])
@pytest.mark.parametrize("op", ["fwd", "inv", "polymul_eval", "polymul", "polymul_bcast"])
def test_limb_split_single_poly(logn, limbs, op):
    """batch == 1 with many limbs runs as limb windows on internal streams
    (run_op split); odd limb counts give a ragged last window."""
    ps, psi = params(logn, limbs)
    p = R.Plan(logn, ps)
    n = 1 << logn
    a = inputs.residues(21, 1, ps, n)
    b = inputs.residues(22, 1, ps, n)
    d = empty_dev(a.shape)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        if op == "fwd":
            R.ntt_forward(p, d, to_dev(a), stream=s)
            want = O.batch(O.OP_FWD, a, ps, psi, n_threads=8)
        elif op == "inv":
            R.ntt_inverse(p, d, to_dev(a), stream=s)
            want = O.batch(O.OP_INV, a, ps, psi, n_threads=8)
        elif op == "polymul_eval":
            bh = O.batch(O.OP_FWD, b, ps, psi, n_threads=8)
            R.polymul(p, d, to_dev(a), to_dev(bh), b_is_eval=True, stream=s)
            want = O.batch(O.OP_POLYMUL, a, ps, psi, b=b, n_threads=8)
        else:
            R.polymul(p, d, to_dev(a), to_dev(b), b_broadcast=(op == "polymul_bcast"), stream=s)
            want = O.batch(O.OP_POLYMUL, a, ps, psi, b=b, n_threads=8)
    s.synchronize()
    assert np.array_equal(from_dev(d), want)


@pytest.mark.parametrize("logn", [4, 5, 7, 9, 10])
@pytest.mark.parametrize("limbs,batch", [(1, 1), (2, 3), (1, 8)])
@pytest.mark.parametrize("op", ["fwd", "inv", "polymul_eval", "polymul", "polymul_bcast"])
def test_latency_path(logn, limbs, batch, op):
    """batch * L <= 8 at N <= 2^10 runs the latency engine k_lat (one CTA per unit)."""
    ps, psi = params(logn, limbs)
    p = R.Plan(logn, ps)
    n = 1 << logn
    a = inputs.residues(51 + logn, batch, ps, n)
    bc = op == "polymul_bcast"
    b = inputs.residues(52 + logn, 1 if bc else batch, ps, n)
    d = empty_dev(a.shape)
    n0 = R.launch_count()
    if op == "fwd":
        R.ntt_forward(p, d, to_dev(a))
        want = O.batch(O.OP_FWD, a, ps, psi)
    elif op == "inv":
        R.ntt_inverse(p, d, to_dev(a))
        want = O.batch(O.OP_INV, a, ps, psi)
    elif op == "polymul_eval":
        bh = O.batch(O.OP_FWD, b, ps, psi)
        R.polymul(p, d, to_dev(a), to_dev(bh), b_is_eval=True)
        want = O.batch(O.OP_POLYMUL, a, ps, psi, b=b)
    else:
        R.polymul(p, d, to_dev(a), to_dev(b), b_broadcast=bc)
        want = O.batch(O.OP_POLYMUL, a, ps, psi, b=b, b_broadcast=bc)
    assert R.launch_count() - n0 == 1
    assert np.array_equal(from_dev(d), want)


# N = 2^10 launch shapes by job size (api.cu launch_warp / lat_units): <= 256 units the
# latency engine, below 3 x 148 x 16 units 4-warp teams, above 2-warp teams -- every mode
# on each shape, ragged batch sizes
@pytest.mark.parametrize("batch", [200, 300, 7200])
@pytest.mark.parametrize("op", ["fwd", "inv", "polymul_eval", "polymul_coeff_bcast"])
def test_n1024_launch_shapes(batch, op):
    ps, psi = params(10, 1)
    p = R.Plan(10, ps)
    a = inputs.residues(61, batch, ps, 1024)
    d = empty_dev(a.shape)
    if op == "fwd":
        R.ntt_forward(p, d, to_dev(a))
        want = O.batch(O.OP_FWD, a, ps, psi, n_threads=8)
    elif op == "inv":
        R.ntt_inverse(p, d, to_dev(a))
        want = O.batch(O.OP_INV, a, ps, psi, n_threads=8)
    elif op == "polymul_eval":
        b = inputs.residues(62, batch, ps, 1024)
        R.polymul(p, d, to_dev(a), to_dev(O.batch(O.OP_FWD, b, ps, psi, n_threads=8)), b_is_eval=True)
        want = O.batch(O.OP_POLYMUL, a, ps, psi, b=b, n_threads=8)
    else:
        b = inputs.residues(63, 1, ps, 1024)
        R.polymul(p, d, to_dev(a), to_dev(b), b_is_eval=False, b_broadcast=True)
        want = O.batch(O.OP_POLYMUL, a, ps, psi, b=b, b_broadcast=True, n_threads=8)
    assert np.array_equal(from_dev(d), want)


@pytest.mark.parametrize("logn", [10, 11, 12, 13, 14, 15, 16])
@pytest.mark.parametrize("limbs,batch", [(1, 1), (2, 1), (1, 2)])
@pytest.mark.parametrize("op", ["fwd", "inv", "polymul_eval", "polymul_bcast"])
def test_cluster_path(logn, limbs, batch, op):
    """batch * L <= 2 at N >= 2^10 runs a single-launch cluster kernel: k_clat
    (ntt_clat.cuh, N <= 2^15) or k_cluster (ntt_cluster.cuh): column stages,
    DSMEM exchange, row stages, exchange, inverse column stages."""
    ps, psi = params(logn, limbs)
    p = R.Plan(logn, ps)
    n = 1 << logn
    a = inputs.residues(41 + logn, batch, ps, n)
    b = inputs.residues(42 + logn, 1 if op == "polymul_bcast" else batch, ps, n)
    d = empty_dev(a.shape)
    n0 = R.launch_count()
    if op == "fwd":
        R.ntt_forward(p, d, to_dev(a))
        want = O.batch(O.OP_FWD, a, ps, psi)
    elif op == "inv":
        R.ntt_inverse(p, d, to_dev(a))
        want = O.batch(O.OP_INV, a, ps, psi)
    else:
        bh = O.batch(O.OP_FWD, b, ps, psi)
        R.polymul(p, d, to_dev(a), to_dev(bh), b_is_eval=True, b_broadcast=(op == "polymul_bcast"))
        want = O.batch(O.OP_POLYMUL, a, ps, psi, b=b, b_broadcast=(op == "polymul_bcast"))
    assert R.launch_count() - n0 == 1          # one launch: the cluster kernel
    assert np.array_equal(from_dev(d), want)


VARIANT_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import inputs, oracle as O, paper_2410_05934_b200 as R
from helpers import params, to_dev, from_dev, empty_dev
ok = True
for logn, limbs, batch in ((10, 1, 37), (10, 2, 5), (16, 3, 2), (13, 2, 3), (16, 9, 1), (12, 8, 1), (11, 2, 1),
                          (14, 1, 2), (4, 2, 9), (5, 1, 7), (6, 1, 5), (7, 2, 3), (8, 1, 9), (9, 1, 5),
                          (16, 64, 3)):
    ps, psi = params(logn, limbs)
    p = R.Plan(logn, ps)
    a = inputs.residues(3, batch, ps, 1 << logn); b = inputs.residues(4, batch, ps, 1 << logn)
    bh = O.batch(O.OP_FWD, b, ps, psi)
    d = empty_dev(a.shape)
    R.ntt_forward(p, d, to_dev(a)); ok &= np.array_equal(from_dev(d), bh * 0 + O.batch(O.OP_FWD, a, ps, psi))
    R.ntt_inverse(p, d, to_dev(bh)); ok &= np.array_equal(from_dev(d), b)
    R.polymul(p, d, to_dev(a), to_dev(bh), b_is_eval=True)
    ok &= np.array_equal(from_dev(d), O.batch(O.OP_POLYMUL_EVAL, a, ps, psi, b=bh))
    R.polymul(p, d, to_dev(a), to_dev(b[:1]), b_broadcast=True)
    ok &= np.array_equal(from_dev(d), O.batch(O.OP_POLYMUL, a, ps, psi, b=b[:1], b_broadcast=True))
print("VARIANT_OK" if ok else "VARIANT_BAD")
"""


@pytest.mark.parametrize("env", [{"RNT_CLUSTER_UNITS": "0"}, {"RNT_CLUSTER_UNITS": "100"},
                                 {"RNT_LAT_UNITS": "0"}, {"RNT_LAT_UNITS": "100000"},
                                 {"RNT_LAZY": "0", "RNT_LAT_UNITS": "0"}, {"RNT_LAZY": "0"},
                                 {"RNT_LAZY": "0", "RNT_CLUSTER_UNITS": "0"}])
def test_kernel_variants(env):
    """Every shipped launch variant (selected by env knobs, read once per process)
    is bit-exact against the oracle."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = VARIANT_SCRIPT.format(root=root, tests=os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env}, capture_output=True, text=True,
                       timeout=600)
    assert "VARIANT_OK" in r.stdout, r.stdout + r.stderr


def test_bench_cfg5_step_exact_inputs():
    """The exact bench.py cfg5 step (its input recipe and launch configuration),
    every output element against the oracle."""
    import importlib.util
    import os

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(root, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    for (logn, limbs, polys, seed) in bench.WORKLOADS["cfg5"]["parts"]:
        mods, a, bhat = bench.make_part_inputs(logn, limbs, polys, seed, 0)
        assert list(mods) == list(params(logn, limbs)[0])  # bench primes == reading C2
        psi = [O.min_psi(q, logn) for q in mods]
        p = R.Plan(logn, mods)
        c = torch.empty(a.shape, dtype=torch.int64, device="cuda")
        R.polymul(p, c, to_dev(a), to_dev(bhat), b_is_eval=True)
        want = O.batch(O.OP_POLYMUL_EVAL, a, mods, psi, b=bhat, n_threads=8)
        assert np.array_equal(from_dev(c), want)


@pytest.mark.parametrize("logn,limbs,batch", [(4, 2, 3), (10, 1, 9), (12, 2, 2), (16, 3, 1)])
def test_automorph_coeff_and_ntt_domain(logn, limbs, batch):
    """rnt_automorph: coefficient form against the oracle definition,
    NTT form against NTT(sigma_g(INTT(A)))."""
    ps, psi = params(logn, limbs)
    p = R.Plan(logn, ps)
    n = 1 << logn
    a = inputs.residues(21, batch, ps, n)
    A = O.batch(O.OP_FWD, a, ps, psi)
    d = empty_dev(a.shape)
    for g in (3, 5, 2 * n - 1, 5 ** 7 % (2 * n)):
        R.automorph(p, d, to_dev(a), g, ntt_domain=False)
        want = np.stack([np.stack([O.automorph(a[b, l], ps[l], g) for l in range(limbs)]) for b in range(batch)])
        assert np.array_equal(from_dev(d), want)
        R.automorph(p, d, to_dev(A), g, ntt_domain=True)
        assert np.array_equal(from_dev(d), O.batch(O.OP_FWD, want, ps, psi))
    with pytest.raises(R.RntError):
        R.automorph(p, d, to_dev(a), 4)          # even Galois element
    x = to_dev(a)
    with pytest.raises(R.RntError):
        R.automorph(p, x, x, 3)                  # aliasing


@pytest.mark.parametrize("logn,n_slot,bg,l", [(10, 37, 20, 3), (10, 64, 30, 2), (10, 5, 10, 6), (6, 50, 20, 3),
                                              (4, 70, 15, 4), (10, 9, 8, 8), (8, 13, 31, 1)])
def test_external_product(logn, n_slot, bg, l):
    """rnt_external_product bit-exact against the oracle, plus the
    gadget-matrix identity c boxtimes G = c."""
    ps, psi = params(logn, 1)
    q, pi = ps[0], psi[0]
    n = 1 << logn
    p = R.Plan(logn, ps)
    c = inputs.residues(31, 2 * n_slot, [q], n).reshape(n_slot, 2, n)
    z = inputs.residues(32, 2 * l * 2, [q], n).reshape(2 * l, 2, n)   # uniform NTT-form key rows
    d = empty_dev(c.shape)
    R.external_product(p, d, to_dev(c), to_dev(z), bg, l)
    got = from_dev(d)
    for s in range(n_slot):
        assert np.array_equal(got[s], O.external_product(c[s], z, q, pi, bg, l))
    # identity with the trivial gadget RGSW (exact decomposition: B^l >= q)
    if (1 << bg) ** l >= q:
        G = np.zeros((2 * l, 2, n), dtype=np.uint64)
        for t in range(2):
            for j in range(l):
                row = np.zeros(n, dtype=np.uint64)
                row[0] = pow(2, bg * j, q)
                G[t * l + j, t] = O.ntt_fwd(row, q, pi)
        R.external_product(p, d, to_dev(c), to_dev(G), bg, l)
        assert np.array_equal(from_dev(d), c)


@pytest.mark.parametrize("logn,L,K,batch", [(16, 12, 13, 1), (10, 5, 4, 7), (4, 3, 2, 5), (12, 45, 3, 2)])
def test_bconv(logn, L, K, batch):
    """rnt_bconv_apply bit-exact against the oracle's BConv."""
    qs = O.primes(logn, L + K)
    src, dst = qs[:L], qs[L:]
    ps = R.Plan(logn, src)
    pd = R.Plan(logn, dst)
    bc = R.BConv(ps, pd)
    x = inputs.residues(41, batch, src, 1 << logn)
    out = empty_dev((batch, K, 1 << logn))
    bc(out, to_dev(x))
    got = from_dev(out)
    for b in range(batch):
        assert np.array_equal(got[b], O.bconv(x[b], src, dst))


def test_bconv_batch_above_grid_limit():
    """batch > 65535 polynomials: the launch is chunked over grid.y."""
    logn, L, K, batch = 4, 2, 1, 70001
    qs = O.primes(logn, L + K)
    src, dst = qs[:L], qs[L:]
    bc = R.BConv(R.Plan(logn, src), R.Plan(logn, dst))
    x = inputs.residues(43, batch, src, 1 << logn)
    out = empty_dev((batch, K, 1 << logn))
    bc(out, to_dev(x))
    got = from_dev(out)
    for b in list(range(0, 40)) + list(range(65500, 65600)) + list(range(batch - 40, batch)):
        assert np.array_equal(got[b], O.bconv(x[b], src, dst))


def test_modup_pipeline_intt_bconv_ntt():
    """CKKS ModUp: NTT-form limbs over Q -> INTT -> BConv -> NTT over P,
    composed from the library calls, against the oracle composition."""
    logn, L, K = 16, 4, 3
    qs = O.primes(logn, L + K)
    src, dst = qs[:L], qs[L:]
    psi_s = [O.min_psi(q, logn) for q in src]
    psi_d = [O.min_psi(q, logn) for q in dst]
    ps, pd = R.Plan(logn, src), R.Plan(logn, dst)
    bc = R.BConv(ps, pd)
    A = inputs.residues(42, 1, src, 1 << logn)              # evaluation form over Q
    coeff = empty_dev(A.shape)
    R.ntt_inverse(ps, coeff, to_dev(A))
    ext = empty_dev((1, K, 1 << logn))
    bc(ext, coeff)
    R.ntt_forward(pd, ext, ext)
    want_c = O.batch(O.OP_INV, A, src, psi_s)
    want = O.batch(O.OP_FWD, O.bconv(want_c[0], src, dst)[None], dst, psi_d)
    assert np.array_equal(from_dev(ext), want)


DEBUG_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import inputs, oracle as O, paper_2410_05934_b200 as R
from helpers import params, to_dev, from_dev, empty_dev
res = []
for logn, limbs, batch in ((10, 2, 3), (16, 2, 1)):
    ps, psi = params(logn, limbs)
    p = R.Plan(logn, ps)
    a = inputs.residues(5, batch, ps, 1 << logn)
    d = empty_dev(a.shape)
    R.ntt_forward(p, d, to_dev(a))                      # canonical: accepted, correct
    res.append(np.array_equal(from_dev(d), O.batch(O.OP_FWD, a, ps, psi)))
    bad = a.copy(); bad[-1, 1, 7] = ps[1]               # r = q_1 in the last limb vector
    for call in (lambda: R.ntt_forward(p, d, to_dev(bad)),
                 lambda: R.ntt_inverse(p, d, to_dev(bad)),
                 lambda: R.pointwise_mul(p, d, to_dev(a), to_dev(bad)),
                 lambda: R.polymul(p, d, to_dev(bad), to_dev(a)),
                 lambda: R.automorph(p, d, to_dev(bad), 3)):
        try:
            call(); torch.cuda.synchronize(); res.append(False)
        except R.RntError as e:
            res.append(e.code == R.RNT_E_INVALID_ARG)
print("DEBUG_OK" if all(res) else "DEBUG_BAD %r" % res)
"""


def test_debug_range_validation():
    """RNT_DEBUG=1: non-canonical residues are rejected with RNT_E_INVALID_ARG
    (reading C6; include/rnsntt.h), canonical inputs still computed exactly."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = DEBUG_SCRIPT.format(root=root, tests=os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, "RNT_DEBUG": "1"}, capture_output=True,
                       text=True, timeout=600)
    assert "DEBUG_OK" in r.stdout, r.stdout + r.stderr


def _primes_below(bits, logn, count):
    """q = 1 (mod 2N) descending from 2^bits (primality from the oracle)."""
    two_n = 2 << logn
    k, out = ((1 << bits) - 1) // two_n, []
    while len(out) < count:
        if O.is_prime(k * two_n + 1):
            out.append(k * two_n + 1)
        k -= 1
    return out


@pytest.mark.parametrize("logn", [4, 7, 8, 10, 11, 13, 16])
@pytest.mark.parametrize("bits", [60, 62])
def test_lazy_ranges(logn, bits):
    """The batched engines (k_warp at > 512 units for N <= 2^10, the column/row
    passes for N >= 2^11) at the extremes of their lazy ranges: 60-bit moduli
    take the LZ kernels (CT reduction only where the bound would pass 16q:
    stages 7, 11, 15), moduli in [2^61, 2^62) the Harvey [0, 4q) kernels.
    Inputs mix all-(q-1), alternating 0 / q-1, deltas and random residues."""
    n = 1 << logn
    ps = _primes_below(bits, logn, 1)
    psi = [O.min_psi(q, logn) for q in ps]
    p = R.Plan(logn, ps)
    q = ps[0]
    B = 640 if logn <= 10 else 8
    a = inputs.residues(77 + logn, B, ps, n)
    a[0::4, 0, :] = q - 1
    a[1::8, 0, :] = np.array([0 if i % 2 else q - 1 for i in range(n)], dtype=np.uint64)
    a[3::8, 0, :] = 0
    a[3::8, 0, 0] = 1
    b = inputs.residues(88 + logn, B, ps, n)
    b[0::3, 0, :] = q - 1
    want = O.batch(O.OP_FWD, a, ps, psi, n_threads=8)
    d = empty_dev(a.shape)
    R.ntt_forward(p, d, to_dev(a))
    assert np.array_equal(from_dev(d), want)
    R.ntt_inverse(p, d, to_dev(want))
    assert np.array_equal(from_dev(d), a)
    bhat = O.batch(O.OP_FWD, b, ps, psi, n_threads=8)
    bhat[1::5, 0, :] = q - 1
    R.polymul(p, d, to_dev(a), to_dev(bhat), b_is_eval=True)
    assert np.array_equal(from_dev(d), O.batch(O.OP_POLYMUL_EVAL, a, ps, psi, b=bhat, n_threads=8))
    R.polymul(p, d, to_dev(a), to_dev(b), b_is_eval=False)
    assert np.array_equal(from_dev(d), O.batch(O.OP_POLYMUL, a, ps, psi, b=b, n_threads=8))


@pytest.mark.parametrize("env", [{"RNT_LAZY": "0"}])
def test_external_product_lazy_off(env):
    """The external product kernels without lazy ranges (RNT_LAZY=0: the CTA kernel at
    N = 2^10, the single-warp kernel below) stay bit-exact."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = f"""
import sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {os.path.join(root, 'tests')!r})
import inputs, oracle as O, paper_2410_05934_b200 as R
from helpers import params, to_dev, from_dev, empty_dev
ok = True
for logn, n_slot, bg, l in ((10, 37, 20, 3), (6, 50, 20, 3)):
    ps, psi = params(logn, 1)
    n = 1 << logn
    p = R.Plan(logn, ps)
    c = inputs.residues(31, 2 * n_slot, ps, n).reshape(n_slot, 2, n)
    z = inputs.residues(32, 2 * l * 2, ps, n).reshape(2 * l, 2, n)
    d = empty_dev(c.shape)
    R.external_product(p, d, to_dev(c), to_dev(z), bg, l)
    got = from_dev(d)
    ok &= all(np.array_equal(got[s], O.external_product(c[s], z, ps[0], psi[0], bg, l)) for s in range(n_slot))
print("EXT_OK" if ok else "EXT_BAD")
"""
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env}, capture_output=True, text=True,
                       timeout=600)
    assert "EXT_OK" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("ws", [3, 8])
def test_sharded_cfg5_on_one_gpu_matches_golden(ws):
    """SURVEY §4.2 T5 on one GPU: the exact ws-way strong split of cfg5 that
    `bench.py --gpus ws` runs (bench.plan_blocks: limb x polynomial shards, inputs
    from global counters), every shard computed by the CUDA path in turn; the
    concatenated per-unit digests equal the oracle's golden hash for the whole job."""
    import importlib.util
    import os

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("rnt_bench_t5", os.path.join(root, "bench.py"))
    B = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(B)
    parts = B.WORKLOADS["cfg5"]["parts"]
    rows = []
    for rank in range(ws):
        for blk in B.plan_blocks(parts, ws, rank, "strong"):
            a, bh = B.block_inputs(blk)
            p = R.Plan(blk["logn"], blk["mods"])
            c = empty_dev(a.shape)
            R.polymul(p, c, to_dev(a), to_dev(bh), b_is_eval=True)
            rows += B.block_digests(blk, from_dev(c))
            p.destroy()
    assert B.check_digests("cfg5", rows) is True
