"""Domain-tagged RNS polynomials over the C ABI (SURVEY 8(b) "Domain tags").

The C ABI is typed by function (rnt_ntt_forward takes coefficient form and
returns NTT form, ...); this module adds SPEC's RnsPoly value type on top of
it, with the Coeff/Eval domain tag and the mismatch errors of S:35-41, S:64-68
and S:156-167:

    a = RnsPoly.from_tensor(plan, t)          # coefficient form, [B][L][N]
    A = forward(a)                            # Eval     (pre Coeff)
    C = pointwise_mul(A, B)                   # Eval     (both Eval, same basis)
    c = inverse(C)                            # Coeff    (incl. N^-1)
    c = polymul(a, b)                         # Coeff    (Eq. 1 end to end)

Errors (all ValueError subclasses, raised on the host before any launch):
    DomainMismatch -- an operand is in the wrong domain, or two operands differ
    BasisMismatch  -- two operands (or an operand and the plan) use different moduli
    PlanMismatch   -- the plan's N differs from the polynomial's N

Every operation runs the library's kernels; nothing here computes residues.
"""
from __future__ import annotations

from dataclasses import dataclass

COEFF = "coeff"
EVAL = "eval"


class DomainMismatch(ValueError):
    pass


class BasisMismatch(ValueError):
    pass


class PlanMismatch(ValueError):
    pass


@dataclass
class RnsPoly:
    """`batch` polynomials of degree < N in the RNS basis `plan.moduli`.

    data: contiguous CUDA tensor (torch.uint64, or torch.int64 as raw 64-bit
    storage) with batch * L * N elements, layout [batch][L][N] (reading C10).
    The polynomial is bound to the plan it was created with; its basis is the
    plan's moduli.
    """
    data: object
    plan: object
    domain: str = COEFF

    def __post_init__(self):
        if self.domain not in (COEFF, EVAL):
            raise ValueError(f"domain must be {COEFF!r} or {EVAL!r}")
        per = self.plan.n_limbs << self.plan.log2n
        if self.data.numel() == 0 or self.data.numel() % per:
            raise PlanMismatch(f"{self.data.numel()} elements is not a whole number of "
                               f"[L={self.plan.n_limbs}][N={1 << self.plan.log2n}] polynomials")

    @classmethod
    def from_tensor(cls, plan, data, domain: str = COEFF) -> "RnsPoly":
        return cls(data, plan, domain)

    @property
    def n(self) -> int:
        return 1 << self.plan.log2n

    @property
    def moduli(self) -> tuple:
        return tuple(int(q) for q in self.plan.moduli)

    @property
    def batch(self) -> int:
        return self.data.numel() // (self.plan.n_limbs << self.plan.log2n)

    def empty_like(self, domain: str | None = None) -> "RnsPoly":
        import torch

        return RnsPoly(torch.empty_like(self.data), self.plan, domain or self.domain)


def _need(p: RnsPoly, domain: str, what: str) -> None:
    if p.domain != domain:
        raise DomainMismatch(f"{what} needs a {domain}-domain polynomial, got {p.domain}")


def _same_basis(a: RnsPoly, b: RnsPoly) -> None:
    if a.n != b.n:
        raise PlanMismatch(f"N differs: {a.n} vs {b.n}")
    if a.moduli != b.moduli:
        raise BasisMismatch("operands are in different RNS bases")


def _same_shape(a: RnsPoly, o: RnsPoly) -> None:
    """`out` must hold exactly a's batch (the kernels write batch * L * N words)."""
    _same_basis(a, o)
    if o.batch != a.batch:
        raise ValueError(f"out batch {o.batch} != operand batch {a.batch}")


def _plan_for(p: RnsPoly, plan):
    if plan is None:
        return p.plan
    if plan.log2n != p.plan.log2n:
        raise PlanMismatch(f"plan N = {1 << plan.log2n}, polynomial N = {p.n}")
    if tuple(int(q) for q in plan.moduli) != p.moduli:
        raise BasisMismatch("plan moduli differ from the polynomial's basis")
    return plan


def _api():
    from . import automorph as _aut
    from . import ntt_forward as _fwd
    from . import ntt_inverse as _inv
    from . import pointwise_mul as _pw
    from . import polymul as _pm
    return _fwd, _inv, _pw, _pm, _aut


def forward(a: RnsPoly, plan=None, out: RnsPoly | None = None, stream=None) -> RnsPoly:
    """NTT^{CT,psi}_{no->bo} (Eq. 1): Coeff -> Eval."""
    _need(a, COEFF, "ntt_forward")
    pl = _plan_for(a, plan)
    o = out if out is not None else a.empty_like(EVAL)
    _same_shape(a, o)
    _api()[0](pl, o.data, a.data, stream=stream)
    o.domain = EVAL
    return o


def inverse(a: RnsPoly, plan=None, out: RnsPoly | None = None, stream=None) -> RnsPoly:
    """INTT^{GS,psi^-1}_{bo->no} incl. N^-1 (Eq. 1): Eval -> Coeff."""
    _need(a, EVAL, "ntt_inverse")
    pl = _plan_for(a, plan)
    o = out if out is not None else a.empty_like(COEFF)
    _same_shape(a, o)
    _api()[1](pl, o.data, a.data, stream=stream)
    o.domain = COEFF
    return o


def pointwise_mul(a: RnsPoly, b: RnsPoly, out: RnsPoly | None = None, stream=None) -> RnsPoly:
    """The (.) of Eq. 1: both Eval, same N and basis; b may be
    a single polynomial broadcast over a's batch."""
    _need(a, EVAL, "pointwise_mul")
    _need(b, EVAL, "pointwise_mul")
    _same_basis(a, b)
    if b.batch not in (1, a.batch):
        raise ValueError(f"batch mismatch: {a.batch} vs {b.batch}")
    o = out if out is not None else a.empty_like(EVAL)
    _same_shape(a, o)
    _api()[2](a.plan, o.data, a.data, b.data, batch=a.batch, b_broadcast=(b.batch != a.batch), stream=stream)
    o.domain = EVAL
    return o


def polymul(a: RnsPoly, b: RnsPoly, out: RnsPoly | None = None, stream=None) -> RnsPoly:
    """c = a b mod (X^N + 1) (Eq. 1 end to end): a in Coeff form; b in Coeff form
    or already in Eval form (reading C8); result in Coeff form."""
    _need(a, COEFF, "polymul")
    _same_basis(a, b)
    if b.batch not in (1, a.batch):
        raise ValueError(f"batch mismatch: {a.batch} vs {b.batch}")
    o = out if out is not None else a.empty_like(COEFF)
    _same_shape(a, o)
    _api()[3](a.plan, o.data, a.data, b.data, b_is_eval=(b.domain == EVAL), batch=a.batch,
              b_broadcast=(b.batch != a.batch), stream=stream)
    o.domain = COEFF
    return o


def automorph(a: RnsPoly, galois_elt: int, out: RnsPoly | None = None, stream=None) -> RnsPoly:
    """sigma_g (Automorph) in the polynomial's own domain."""
    if galois_elt % 2 == 0:
        raise ValueError("Galois element must be odd")
    o = out if out is not None else a.empty_like()
    _same_shape(a, o)
    _api()[4](a.plan, o.data, a.data, galois_elt, ntt_domain=(a.domain == EVAL), batch=a.batch, stream=stream)
    o.domain = a.domain
    return o
