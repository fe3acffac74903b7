"""Shared test helpers: device upload/download of uint64 arrays (stored in
torch.int64 tensors as raw 64-bit words) and oracle-side parameter sets."""
from __future__ import annotations

import functools

import numpy as np

import oracle as O


def to_dev(a: np.ndarray, device="cuda"):
    import torch

    a = np.ascontiguousarray(a, dtype=np.uint64)
    return torch.from_numpy(a.view(np.int64).copy()).to(device)


def from_dev(t) -> np.ndarray:
    return t.detach().cpu().numpy().view(np.uint64)


def empty_dev(shape, device="cuda"):
    import torch

    return torch.empty(shape, dtype=torch.int64, device=device)


@functools.lru_cache(maxsize=None)
def params(logn: int, limbs: int):
    """Reading C2 primes and reading C1 psi, from the oracle."""
    ps = O.primes(logn, limbs)
    psi = [O.min_psi(q, logn) for q in ps]
    return tuple(ps), tuple(psi)
