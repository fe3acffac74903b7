"""Seeded synthetic input generator shared by the oracle tests, the GPU parity
tests and bench.py.

It holds none of the method's arithmetic: only a counter-based SplitMix64
stream and the Lemire multiply-shift map of a 64-bit word onto [0, q).  Inputs
are uniform residues, the distribution of RLWE ciphertext polynomials (the
"A(x)" of a ciphertext is uniform mod Q); limbs are independent
draws (reading C11).

    z   = splitmix64(seed, ctr)          ctr = (b * L + l) * N + i
    res = (z * q) >> 64                  (Lemire multiply-shift)

Operand a uses the config seed; operand b uses seed + 1.
"""
from __future__ import annotations

import numpy as np

_M32 = np.uint64(0xFFFFFFFF)
_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, ctr: np.ndarray) -> np.ndarray:
    """z = seed + (ctr + 1) * golden; two xor-shift-multiply rounds (mod 2^64)."""
    ctr = np.asarray(ctr, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + (ctr + np.uint64(1)) * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
        z = z ^ (z >> np.uint64(31))
    return z


def _mulhi64(z: np.ndarray, q: int) -> np.ndarray:
    qh, ql = np.uint64(q >> 32), np.uint64(q & 0xFFFFFFFF)
    zh, zl = z >> np.uint64(32), z & _M32
    with np.errstate(over="ignore"):
        ll = zl * ql
        lh = zl * qh
        hl = zh * ql
        hh = zh * qh
        mid = (ll >> np.uint64(32)) + (lh & _M32) + (hl & _M32)
        return hh + (lh >> np.uint64(32)) + (hl >> np.uint64(32)) + (mid >> np.uint64(32))


def residues(seed: int, batch: int, moduli, n: int, batch_offset: int = 0) -> np.ndarray:
    """[batch][L][n] uint64 uniform residues; limb l is reduced into [0, moduli[l]).

    `batch_offset` shifts the polynomial index used in the counter, so a shard
    of polynomials [o, o + batch) of a larger global batch reproduces exactly
    the same values as the global array (multi-GPU sharding).
    """
    L = len(moduli)
    out = np.empty((batch, L, n), dtype=np.uint64)
    i = np.arange(n, dtype=np.uint64)
    for b in range(batch):
        for l, q in enumerate(moduli):
            ctr = np.uint64(((batch_offset + b) * L + l) * n) + i
            out[b, l] = _mulhi64(splitmix64(seed, ctr), int(q))
    return out


def residues_limbs(seed: int, batch: int, moduli, n: int, limb_offset: int, total_limbs: int,
                   batch_offset: int = 0) -> np.ndarray:
    """Like `residues`, for the limb slice [limb_offset, limb_offset + len(moduli))
    of a global [*][total_limbs][n] array (counters use the global limb index)."""
    L = len(moduli)
    out = np.empty((batch, L, n), dtype=np.uint64)
    i = np.arange(n, dtype=np.uint64)
    for b in range(batch):
        for l, q in enumerate(moduli):
            ctr = np.uint64(((batch_offset + b) * total_limbs + limb_offset + l) * n) + i
            out[b, l] = _mulhi64(splitmix64(seed, ctr), int(q))
    return out


def digest(x: np.ndarray) -> tuple[int, int]:
    """(sum, weighted sum) of a vector mod 2^64: sum x_i, sum (i+1) x_i."""
    x = np.asarray(x, dtype=np.uint64).ravel()
    w = np.arange(1, x.size + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return int(np.sum(x, dtype=np.uint64)), int(np.sum(x * w, dtype=np.uint64))
