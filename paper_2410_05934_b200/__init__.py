"""B200-native batched negacyclic NTT / INTT / polymul in RNS form.

Thin ctypes binding over librnsntt.so (C ABI: include/rnsntt.h).  Every step
of the path runs in the library's sm_100a kernels; this module only
marshals arguments.  There is no CPU fallback: importing the package on a
box without the built library raises immediately.

Functions keep the C names without the ``rnt_`` prefix:

    plan = Plan(log2n, moduli, psi=None, device=0)
    ntt_forward(plan, out, inp)             # NTT^{CT,psi}_{no->bo}  (Eq. 1)
    ntt_inverse(plan, out, inp)             # INTT^{GS,psi^-1}_{bo->no} incl. N^{-1}
    pointwise_mul(plan, c, a_hat, b_hat)    # the (.) of Eq. 1
    polymul(plan, c, a, b, b_is_eval=False) # Eq. 1 end to end

Tensors are CUDA tensors of dtype torch.uint64 (or torch.int64 used as raw
64-bit storage), contiguous, shaped [batch, n_limbs, N] (or any shape with
batch*n_limbs*N elements; batch is inferred).
"""
from __future__ import annotations

import ctypes
import os

from . import _lib
from ._lib import (RNT_E_CUDA, RNT_E_INVALID_ARG, RNT_E_MODULUS, RNT_E_OOM, RNT_E_PLAN_MISMATCH,
                   RNT_E_ROOT, RNT_E_UNSUPPORTED_N, RNT_OK, RntError, launch_count, lib_path,
                   status_string)

__all__ = [
    "Plan", "BConv", "KeySwitch", "ntt_forward", "ntt_inverse", "pointwise_mul", "polymul", "automorph", "external_product",
    "hrf_matvec", "execute_host",
    "RntError", "status_string", "launch_count", "lib_path",
    "RNT_OK", "RNT_E_INVALID_ARG", "RNT_E_UNSUPPORTED_N", "RNT_E_MODULUS", "RNT_E_ROOT",
    "RNT_E_PLAN_MISMATCH", "RNT_E_CUDA", "RNT_E_OOM",
    "OP_FORWARD", "OP_INVERSE", "OP_POLYMUL_EVAL", "OP_POLYMUL",
    "rnt_ntt_forward", "rnt_ntt_inverse", "rnt_pointwise_mul", "rnt_polymul", "rnt_automorph",
    "rnt_external_product", "rnt_hrf_matvec", "rnt_execute_host",
    "rnt_status_string", "rnt_launch_count",
]

OP_FORWARD, OP_INVERSE, OP_POLYMUL_EVAL, OP_POLYMUL = 0, 1, 2, 3


class Plan:
    """rnt_plan: N = 2^log2n, one ~60-bit NTT-friendly prime per limb."""

    def __init__(self, log2n: int, moduli, psi=None, device: int | None = None):
        if device is None:
            import torch

            device = torch.cuda.current_device() if torch.cuda.is_available() else 0
        mods = [int(m) for m in moduli]
        L = len(mods)
        marr = (ctypes.c_uint64 * max(L, 1))(*mods)
        parr = None
        if psi is not None:
            ps = [int(x) for x in psi]
            if len(ps) != L:
                raise ValueError("psi must have one entry per modulus")
            parr = (ctypes.c_uint64 * L)(*ps)
        h = ctypes.c_void_p()
        _lib.check(_lib.L.rnt_plan_create(ctypes.byref(h), log2n, L, marr, parr, device))
        self._h = h
        self.log2n = log2n
        self.n = 1 << log2n
        self.n_limbs = L
        self.moduli = mods
        self.device = device

    @property
    def handle(self):
        if self._h is None:
            raise RntError(RNT_E_INVALID_ARG, "plan destroyed")
        return self._h

    def psi(self):
        out = (ctypes.c_uint64 * self.n_limbs)()
        _lib.check(_lib.L.rnt_plan_query(self.handle, None, None, out, None))
        return [int(v) for v in out]

    def destroy(self):
        if getattr(self, "_h", None) is not None:
            _lib.L.rnt_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.destroy()


def _ptr(t, plan: Plan | None = None, need: int | None = None, what: str = "tensor") -> int:
    """Device pointer of a contiguous CUDA tensor of 64-bit words, checked against
    the words the call will touch (`need`) and the plan's device; an int is taken
    as a raw device address (the caller vouches for it)."""
    if hasattr(t, "data_ptr"):
        if not t.is_cuda or not t.is_contiguous():
            raise ValueError(f"{what}: expected a contiguous CUDA tensor")
        if t.element_size() != 8:
            raise ValueError(f"{what}: expected 64-bit elements (torch.uint64 / torch.int64), got {t.dtype}")
        if plan is not None and t.device.index != plan.device:
            raise ValueError(f"{what}: on cuda:{t.device.index}, plan is on cuda:{plan.device}")
        if need is not None and t.numel() < need:
            raise ValueError(f"{what}: {t.numel()} elements, the call needs {need}")
        return t.data_ptr()
    return int(t)


def _host_ptr(t, need: int | None = None, what: str = "host tensor") -> int:
    if hasattr(t, "data_ptr"):
        if t.is_cuda or not t.is_contiguous() or t.element_size() != 8:
            raise ValueError(f"{what}: expected a contiguous host tensor of 64-bit elements")
        if need is not None and t.numel() < need:
            raise ValueError(f"{what}: {t.numel()} elements, the call needs {need}")
        return t.data_ptr()
    return int(t)


def _batch(plan: Plan, t, batch):
    if batch is not None:
        return int(batch)
    per = plan.n_limbs * plan.n
    numel = t.numel()
    if numel % per:
        raise ValueError(f"tensor of {numel} elements is not a whole number of [L={plan.n_limbs}][N={plan.n}] polynomials")
    return numel // per


def _stream(stream) -> int | None:
    if stream is None:
        import torch

        return torch.cuda.current_stream().cuda_stream
    if hasattr(stream, "cuda_stream"):
        return stream.cuda_stream
    return int(stream)


def ntt_forward(plan: Plan, out, inp, batch=None, stream=None) -> None:
    """NTT^{CT,psi}_{no->bo} of every limb of every polynomial (Eq. 1)."""
    b = _batch(plan, inp, batch)
    w = b * plan.n_limbs * plan.n
    _lib.check(_lib.L.rnt_ntt_forward(plan.handle, _ptr(out, plan, w, "out"), _ptr(inp, plan, w, "inp"), b,
                                      _stream(stream)))


def ntt_inverse(plan: Plan, out, inp, batch=None, stream=None) -> None:
    """INTT^{GS,psi^-1}_{bo->no} including N^{-1} (Eq. 1)."""
    b = _batch(plan, inp, batch)
    w = b * plan.n_limbs * plan.n
    _lib.check(_lib.L.rnt_ntt_inverse(plan.handle, _ptr(out, plan, w, "out"), _ptr(inp, plan, w, "inp"), b,
                                      _stream(stream)))


def _b_words(plan: Plan, b: int, broadcast: bool) -> int:
    return plan.n_limbs * plan.n * (1 if broadcast else b)


def pointwise_mul(plan: Plan, c, a_hat, b_hat, batch=None, b_broadcast=False, stream=None) -> None:
    """c = a_hat (.) b_hat mod q_l (NTT domain)."""
    b = _batch(plan, a_hat, batch)
    w = b * plan.n_limbs * plan.n
    _lib.check(_lib.L.rnt_pointwise_mul(plan.handle, _ptr(c, plan, w, "c"), _ptr(a_hat, plan, w, "a_hat"),
                                        _ptr(b_hat, plan, _b_words(plan, b, b_broadcast), "b_hat"), b,
                                        int(bool(b_broadcast)), _stream(stream)))


def polymul(plan: Plan, c, a, b_op, b_is_eval=False, batch=None, b_broadcast=False, stream=None) -> None:
    """c = a * b mod (x^N + 1) per limb via Eq. 1 (b_op in NTT form if b_is_eval)."""
    b = _batch(plan, a, batch)
    w = b * plan.n_limbs * plan.n
    _lib.check(_lib.L.rnt_polymul(plan.handle, _ptr(c, plan, w, "c"), _ptr(a, plan, w, "a"),
                                  _ptr(b_op, plan, _b_words(plan, b, b_broadcast), "b"), b, int(bool(b_is_eval)),
                                  int(bool(b_broadcast)), _stream(stream)))


def automorph(plan: Plan, out, inp, galois_elt: int, ntt_domain: bool = True, batch=None, stream=None) -> None:
    """sigma_g: a(x) -> a(x^g) mod (x^N+1) (Automorph); NTT form is a slot permutation."""
    b = _batch(plan, inp, batch)
    w = b * plan.n_limbs * plan.n
    _lib.check(_lib.L.rnt_automorph(plan.handle, _ptr(out, plan, w, "out"), _ptr(inp, plan, w, "inp"), b,
                                    int(galois_elt), int(bool(ntt_domain)), _stream(stream)))


def external_product(plan: Plan, out, c, rgsw_hat, base_log2: int, levels: int, n_slot=None,
                     stream=None) -> None:
    """TFHE external product of n_slot RLWE pairs with one RGSW key in NTT form
    (CMux-level batching P:324-332): out, c [n_slot][2][N]; rgsw_hat [2l][2][N]."""
    ns = int(n_slot) if n_slot is not None else c.numel() // (2 * plan.n)
    w = ns * 2 * plan.n
    _lib.check(_lib.L.rnt_external_product(plan.handle, _ptr(out, plan, w, "out"), _ptr(c, plan, w, "c"),
                                           _ptr(rgsw_hat, plan, 4 * int(levels) * plan.n, "rgsw_hat"), ns,
                                           int(base_log2), int(levels), _stream(stream)))


def hrf_matvec(plan: Plan, out, pt, ct, n_slot=None, add=None, stream=None) -> None:
    """HRF-MatVec of repack (tab:repack), NTT form:
    out[c][l] = add[c][l] + sum_j pt[j][l] (.) ct[j][c][l].
    out, add [2][L][N]; pt [n_slot][L][N]; ct [n_slot][2][L][N]; add may be out."""
    ln = plan.n_limbs * plan.n
    ns = int(n_slot) if n_slot is not None else pt.numel() // ln
    _lib.check(_lib.L.rnt_hrf_matvec(plan.handle, _ptr(out, plan, 2 * ln, "out"),
                                     _ptr(pt, plan, ns * ln, "pt") if ns else None,
                                     _ptr(ct, plan, 2 * ns * ln, "ct") if ns else None, ns,
                                     _ptr(add, plan, 2 * ln, "add") if add is not None else None,
                                     _stream(stream)))


class BConv:
    """Fast basis conversion Q (plan `src`) -> P (plan `dst`) (BConv)."""

    def __init__(self, src: Plan, dst: Plan):
        h = ctypes.c_void_p()
        _lib.check(_lib.L.rnt_bconv_create(ctypes.byref(h), src.handle, dst.handle))
        self._h = h
        self.src, self.dst = src, dst

    def __call__(self, out, inp, batch=None, stream=None) -> None:
        b = int(batch) if batch is not None else _batch(self.src, inp, None)
        _lib.check(_lib.L.rnt_bconv_apply(self._h, _ptr(out, self.dst, b * self.dst.n_limbs * self.dst.n, "out"),
                                          _ptr(inp, self.src, b * self.src.n_limbs * self.src.n, "inp"), b,
                                          _stream(stream)))

    def destroy(self):
        if getattr(self, "_h", None) is not None:
            _lib.L.rnt_bconv_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


class KeySwitch:
    """CKKS hybrid key switching (rnt_keyswitch_*).

    q_plan: basis Q (L limbs); qp_plan: Q followed by the special primes P;
    dnum digits of ceil(L / dnum) primes.  __call__(out [2][L][N], d [L][N],
    evk [dnum][2][L+K][N], add0 [L][N] or None), all NTT form.
    """

    def __init__(self, q_plan: Plan, qp_plan: Plan, dnum: int):
        h = ctypes.c_void_p()
        _lib.check(_lib.L.rnt_keyswitch_create(ctypes.byref(h), q_plan.handle, qp_plan.handle, int(dnum)))
        self._h = h
        self.q_plan, self.qp_plan, self.dnum = q_plan, qp_plan, int(dnum)
        a = ctypes.c_uint32()
        wb = ctypes.c_uint64()
        _lib.check(_lib.L.rnt_keyswitch_query(h, ctypes.byref(a), ctypes.byref(wb)))
        self.alpha, self.workspace_bytes = int(a.value), int(wb.value)

    def __call__(self, out, d, evk, add0=None, stream=None) -> None:
        qp, qpp = self.q_plan, self.qp_plan
        ln = qp.n_limbs * qp.n
        _lib.check(_lib.L.rnt_keyswitch_apply(
            self._h, _ptr(out, qp, 2 * ln, "out"), _ptr(d, qp, ln, "d"),
            _ptr(evk, qp, self.dnum * 2 * qpp.n_limbs * qpp.n, "evk"),
            _ptr(add0, qp, ln, "add0") if add0 is not None else None, _stream(stream)))

    def destroy(self):
        if getattr(self, "_h", None) is not None:
            _lib.L.rnt_keyswitch_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def execute_host(plan: Plan, op: int, out_host, in_host, dev_ws, b_dev=None, batch=None,
                 b_broadcast=False, stream=None) -> None:
    """Host buffers in/out (pinned recommended): H2D copy, op, D2H copy, async."""
    hb = _batch(plan, in_host, batch)
    w = hb * plan.n_limbs * plan.n
    bptr = _ptr(b_dev, plan, _b_words(plan, hb, b_broadcast), "b_dev") if b_dev is not None else None
    _lib.check(_lib.L.rnt_execute_host(plan.handle, int(op), _host_ptr(out_host, w, "out_host"),
                                       _host_ptr(in_host, w, "in_host"), _ptr(dev_ws, plan, w, "dev_ws"), bptr, hb,
                                       int(bool(b_broadcast)), _stream(stream)))


# Aliases with the exact C-ABI names (include/rnsntt.h).
rnt_ntt_forward = ntt_forward
rnt_ntt_inverse = ntt_inverse
rnt_pointwise_mul = pointwise_mul
rnt_polymul = polymul
rnt_automorph = automorph
rnt_external_product = external_product
rnt_hrf_matvec = hrf_matvec
rnt_execute_host = execute_host
rnt_status_string = status_string
rnt_launch_count = launch_count


# Domain-tagged polynomial layer: RnsPoly + mismatch errors.
from . import poly  # noqa: E402
from .poly import COEFF, EVAL, BasisMismatch, DomainMismatch, PlanMismatch, RnsPoly  # noqa: E402

__all__ += ["poly", "RnsPoly", "COEFF", "EVAL", "DomainMismatch", "BasisMismatch", "PlanMismatch"]
