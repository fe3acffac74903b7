"""CPU oracle for the batched negacyclic NTT / INTT / pointwise path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_2410_05934_b200`` never imports it, and
the two share no code: the oracle is plain C (``ntt_oracle.c``) with exact
128-bit ``%`` arithmetic, compiled here with gcc and called through ctypes.

Every function cites the passage it follows (P:n = PAPER.md line n,
S:n = SPEC.md line n); see ``ntt_oracle.c`` for the arithmetic.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ntt_oracle.c")
_HDR = os.path.join(_HERE, "ntt_oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

_u64p = ctypes.POINTER(ctypes.c_uint64)


def build(force: bool = False) -> str:
    """Compile ntt_oracle.c into liboracle.so (gcc -O2, pthreads)."""
    newest = max(os.path.getmtime(_SRC), os.path.getmtime(_HDR))
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < newest:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread", "-o", tmp, _SRC]
        )
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            u64, u32, i32 = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int
            sig = {
                "or_mulmod": (u64, [u64, u64, u64]),
                "or_addmod": (u64, [u64, u64, u64]),
                "or_submod": (u64, [u64, u64, u64]),
                "or_powmod": (u64, [u64, u64, u64]),
                "or_is_prime": (i32, [u64]),
                "or_brv": (u32, [u32, u32]),
                "or_is_primitive_2n_root": (i32, [u64, u64, u32]),
                "or_min_psi": (u64, [u64, u32]),
                "or_primes": (i32, [u32, u32, _u64p]),
                "or_tables": (None, [u64, u64, u32, _u64p, _u64p, _u64p]),
                "or_ntt_fwd": (None, [_u64p, u32, u64, _u64p]),
                "or_ntt_inv": (None, [_u64p, u32, u64, _u64p, u64]),
                "or_pointwise": (None, [_u64p, _u64p, _u64p, u64, u64]),
                "or_naive_ntt_at": (u64, [_u64p, u32, u64, u64, u32]),
                "or_naive_ntt": (None, [_u64p, _u64p, u32, u64, u64]),
                "or_naive_intt_at": (u64, [_u64p, u32, u64, u64, u32]),
                "or_schoolbook_at": (u64, [_u64p, _u64p, u32, u64, u32]),
                "or_schoolbook": (None, [_u64p, _u64p, _u64p, u32, u64]),
                "or_automorph": (None, [_u64p, _u64p, u32, u64, u64]),
                "or_decompose": (None, [_u64p, u64, u64, u32, u32]),
                "or_external_product": (None, [_u64p, _u64p, _u64p, u32, u64, u64, u32, u32]),
                "or_bconv": (None, [_u64p, _u64p, u64, _u64p, u32, _u64p, u32]),
                "or_hrf_matvec": (None, [_u64p, _u64p, _u64p, _u64p, u32, _u64p, u32, u64]),
                "or_keyswitch": (None, [_u64p, _u64p, _u64p, _u64p, u32, _u64p, u32, _u64p, u32, u32]),
                "or_batch": (i32, [i32, _u64p, _u64p, i32, u32, u32, u32, _u64p, _u64p, i32]),
            }
            for name, (res, args) in sig.items():
                f = getattr(lib, name)
                f.restype = res
                f.argtypes = args
            _lib = lib
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.uint64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_u64p)


def _vec(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def _check_canonical(a: np.ndarray, q: int) -> None:
    # Reading C6: residues must be canonical in [0, q).
    if a.size and int(a.max()) >= q:
        raise ValueError("residue >= q (precondition C6)")


# ------------------------------------------------------------------ scalars
def mulmod(a: int, b: int, q: int) -> int:
    return int(_load().or_mulmod(a, b, q))


def powmod(b: int, e: int, q: int) -> int:
    return int(_load().or_powmod(b, e, q))


def is_prime(n: int) -> bool:
    return bool(_load().or_is_prime(n))


def brv(i: int, logn: int) -> int:
    return int(_load().or_brv(i, logn))


def is_primitive_2n_root(psi: int, q: int, logn: int) -> bool:
    """psi^{2N} = 1 and psi^i != 1 for 0 < i < 2N."""
    return bool(_load().or_is_primitive_2n_root(psi, q, logn))


def min_psi(q: int, logn: int) -> int:
    """Reading C1: the numerically smallest primitive 2N-th root of unity."""
    return int(_load().or_min_psi(q, logn))


def primes(logn: int, count: int) -> list[int]:
    """Reading C2: the `count` largest primes q < 2^60 with q = 1 mod 2N."""
    out = np.zeros(count, dtype=np.uint64)
    if _load().or_primes(logn, count, _p(out)) != 0:
        raise ValueError("not enough primes")
    return [int(x) for x in out]


def tables(q: int, psi: int, logn: int):
    """fwd[i] = psi^{brv(i)}, inv[i] = psi^{-brv(i)}, N^{-1} mod q."""
    n = 1 << logn
    fwd = np.zeros(n, dtype=np.uint64)
    inv = np.zeros(n, dtype=np.uint64)
    ninv = np.zeros(1, dtype=np.uint64)
    _load().or_tables(q, psi, logn, _p(fwd), _p(inv), _p(ninv))
    return fwd, inv, int(ninv[0])


# --------------------------------------------------------------- transforms
def ntt_fwd(a, q: int, psi: int) -> np.ndarray:
    """NTT^{CT,psi}_{no->bo}(a) of Eq. 1; returns a new array."""
    a = _vec(a).copy()
    logn = int(a.size).bit_length() - 1
    _check_canonical(a, q)
    fwd, _, _ = tables(q, psi, logn)
    _load().or_ntt_fwd(_p(a), logn, q, _p(fwd))
    return a


def ntt_inv(A, q: int, psi: int) -> np.ndarray:
    """INTT^{GS,psi^-1}_{bo->no}(A) of Eq. 1 including x N^{-1}."""
    A = _vec(A).copy()
    logn = int(A.size).bit_length() - 1
    _check_canonical(A, q)
    _, inv, ninv = tables(q, psi, logn)
    _load().or_ntt_inv(_p(A), logn, q, _p(inv), ninv)
    return A


def pointwise(a, b, q: int) -> np.ndarray:
    """The (.) of Eq. 1: c_k = a_k b_k mod q."""
    a, b = _vec(a), _vec(b)
    c = np.zeros_like(a)
    _load().or_pointwise(_p(c), _p(a), _p(b), a.size, q)
    return c


def naive_ntt(a, q: int, psi: int) -> np.ndarray:
    """Definition: NTT(a)[k] = sum_i a_i psi^{(2 brv(k)+1) i} (O(N^2))."""
    a = _vec(a)
    logn = int(a.size).bit_length() - 1
    out = np.zeros_like(a)
    _load().or_naive_ntt(_p(out), _p(a), logn, q, psi)
    return out


def naive_ntt_at(a, q: int, psi: int, k: int) -> int:
    a = _vec(a)
    return int(_load().or_naive_ntt_at(_p(a), int(a.size).bit_length() - 1, q, psi, k))


def naive_intt_at(A, q: int, psi: int, i: int) -> int:
    A = _vec(A)
    return int(_load().or_naive_intt_at(_p(A), int(A.size).bit_length() - 1, q, psi, i))


def schoolbook(a, b, q: int) -> np.ndarray:
    """c = a b mod (x^N + 1), O(N^2)."""
    a, b = _vec(a), _vec(b)
    c = np.zeros_like(a)
    _load().or_schoolbook(_p(c), _p(a), _p(b), int(a.size).bit_length() - 1, q)
    return c


def schoolbook_at(a, b, q: int, k: int) -> int:
    a, b = _vec(a), _vec(b)
    return int(_load().or_schoolbook_at(_p(a), _p(b), int(a.size).bit_length() - 1, q, k))


def automorph(a, q: int, g: int) -> np.ndarray:
    """sigma_g(a)(x) = a(x^g) mod (x^N + 1), g odd (Automorph)."""
    a = _vec(a)
    out = np.zeros_like(a)
    _load().or_automorph(_p(out), _p(a), int(a.size).bit_length() - 1, q, g)
    return out


def decompose(v: int, q: int, base_log2: int, levels: int) -> list[int]:
    """Signed gadget digits of v mod q as residues (Decompose)."""
    out = np.zeros(levels, dtype=np.uint64)
    _load().or_decompose(_p(out), v, q, base_log2, levels)
    return [int(x) for x in out]


def external_product(c, rgsw_hat, q: int, psi: int, base_log2: int, levels: int) -> np.ndarray:
    """TFHE external product: c [2][N], rgsw_hat [2l][2][N] (NTT form) -> [2][N]."""
    c = np.ascontiguousarray(c, dtype=np.uint64)
    z = np.ascontiguousarray(rgsw_hat, dtype=np.uint64)
    n = c.shape[-1]
    assert c.shape == (2, n) and z.shape == (2 * levels, 2, n)
    _check_canonical(c, q)
    out = np.zeros_like(c)
    _load().or_external_product(_p(out), _p(c), _p(z), n.bit_length() - 1, q, psi, base_log2, levels)
    return out


def hrf_matvec(pt, ct, moduli, add=None) -> np.ndarray:
    """HRF-MatVec (tab:repack): out[c][l] = add[c][l] + sum_j pt[j][l] (.) ct[j][c][l]
    mod q_l, NTT form.  pt [n_slot][L][N], ct [n_slot][2][L][N], add [2][L][N] or None."""
    pt = np.ascontiguousarray(pt, dtype=np.uint64)
    ct = np.ascontiguousarray(ct, dtype=np.uint64)
    ns, L, n = pt.shape
    assert ct.shape == (ns, 2, L, n)
    qs = _vec(moduli)
    assert qs.size == L
    for l in range(L):
        _check_canonical(pt[:, l], int(qs[l]))
        _check_canonical(ct[:, :, l], int(qs[l]))
    a = None
    if add is not None:
        a = np.ascontiguousarray(add, dtype=np.uint64)
        assert a.shape == (2, L, n)
        for l in range(L):
            _check_canonical(a[:, l], int(qs[l]))
    out = np.zeros((2, L, n), dtype=np.uint64)
    _load().or_hrf_matvec(_p(out), _p(pt), _p(ct), _p(a) if a is not None else None, ns, _p(qs), L, n)
    return out


def bconv(x, q_basis, p_basis) -> np.ndarray:
    """Fast basis conversion Q -> P (BConv): x [L][N] -> [K][N]."""
    x = np.ascontiguousarray(x, dtype=np.uint64)
    L, n = x.shape
    qs, ps = _vec(q_basis), _vec(p_basis)
    assert qs.size == L
    for i in range(L):
        _check_canonical(x[i], int(qs[i]))
    out = np.zeros((ps.size, n), dtype=np.uint64)
    _load().or_bconv(_p(out), _p(x), n, _p(qs), L, _p(ps), ps.size)
    return out


def keyswitch(d, evk, q_basis, p_basis, dnum: int, add0=None) -> np.ndarray:
    """CKKS hybrid key switching (f2; readings KS1-KS4):
    d [L][N] and evk [dnum][2][L+K][N] in NTT form -> out [2][L][N] NTT form over Q."""
    d = np.ascontiguousarray(d, dtype=np.uint64)
    L, n = d.shape
    qs, ps = _vec(q_basis), _vec(p_basis)
    K = ps.size
    assert qs.size == L and 1 <= dnum <= L
    alpha = -(-L // dnum)
    if (dnum - 1) * alpha >= L:
        raise ValueError("empty digit: (dnum - 1) * ceil(L / dnum) >= L")
    z = np.ascontiguousarray(evk, dtype=np.uint64)
    assert z.shape == (dnum, 2, L + K, n)
    for i in range(L):
        _check_canonical(d[i], int(qs[i]))
    a0 = None
    if add0 is not None:
        a0 = np.ascontiguousarray(add0, dtype=np.uint64)
        assert a0.shape == (L, n)
    out = np.zeros((2, L, n), dtype=np.uint64)
    _load().or_keyswitch(_p(out), _p(d), _p(z), _p(a0) if a0 is not None else None, n.bit_length() - 1,
                         _p(qs), L, _p(ps), K, dnum)
    return out


# -------------------------------------------------------------------- batch
OP_FWD, OP_INV, OP_POLYMUL_EVAL, OP_POLYMUL = 0, 1, 2, 3


def batch(op: int, data: np.ndarray, moduli, psi, b: np.ndarray | None = None,
          b_broadcast: bool = False, n_threads: int = 1) -> np.ndarray:
    """Apply `op` to every (batch, limb) unit of a [B][L][N] uint64 array.

    op: OP_FWD, OP_INV, OP_POLYMUL_EVAL (c = INTT(NTT(a) . b_hat)) or
    OP_POLYMUL (c = INTT(NTT(a) . NTT(b))).  Returns a new array; the input is
    not modified.  Layout per reading C10.
    """
    data = np.ascontiguousarray(data, dtype=np.uint64).copy()
    assert data.ndim == 3
    B, L, N = data.shape
    logn = N.bit_length() - 1
    mod = _vec(moduli)
    ps = _vec(psi)
    assert mod.size == L and ps.size == L
    for l in range(L):
        _check_canonical(data[:, l, :], int(mod[l]))
    bp = None
    if op in (OP_POLYMUL_EVAL, OP_POLYMUL):
        b = np.ascontiguousarray(b, dtype=np.uint64)
        assert b.shape == ((1 if b_broadcast else B), L, N)
        bp = _p(b)
    else:
        b_broadcast = False
    rc = _load().or_batch(op, _p(data), bp, int(b_broadcast), B, L, logn, _p(mod), _p(ps),
                          int(n_threads))
    assert rc == 0
    return data
