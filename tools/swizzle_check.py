"""Bank-conflict check of warp-buffer layouts for the warp engine (ntt_small.cuh):
the shipped padding phys(j) = j + (j >> 4) and a conflict-free XOR swizzle
(measured 2 % slower in k_warp: ptxas spends fmaheavy IMADs on the address
XORs; KB1).

Shared memory has 32 four-byte banks; a 64-bit access of a half-warp (16
lanes) is conflict-free when the 16 word addresses fall into 16 distinct bank
pairs (word mod 16).  For every pass of every warp-engine schedule (N = 2^4 ..
2^10 split-tail radix-8 and the rows' radix-8 schedule) this enumerates the
addresses each half-warp touches for every group element and reports the
wavefronts against the ideal (one per half-warp access).

    python tools/swizzle_check.py
"""
from __future__ import annotations


def swz_low(j: int) -> int:            # j4 -> 0101, j5 -> 1010, j6 -> 1100 into the bank bits
    return (((j >> 4) & 1) * 5) ^ (((j >> 5) & 1) * 10) ^ (((j >> 6) & 1) * 12)


def wswz(j: int) -> int:
    return j ^ swz_low(j)


def pad(j: int) -> int:                # the round-1 layout, for comparison
    return j + (j >> 4)


def passes(logn: int, km: int):
    b = km // 10 if km >= 10 else km
    n_p = (logn + b - 1) // b
    split = km >= 10 and n_p >= 2 and logn - b * (n_p - 1) == 1 and b >= 3

    def k(p):
        if split:
            return b if p < n_p - 2 else (b - 1 if p == n_p - 2 else 2)
        return b if p < n_p - 1 else logn - b * (n_p - 1)

    def s(p):
        return b * (n_p - 2) + b - 1 if (split and p == n_p - 1) else p * b
    return [(s(p), k(p)) for p in range(n_p)]


def accesses(logn: int, s: int, k: int):
    n, r = 1 << logn, 1 << k
    lo = 1 << (logn - s - k)
    gpp = n // r
    gpl = (1024 // r) // 32
    for gi in range(gpl):
        for i in range(r):
            out = []
            for lane in range(32):
                g = lane + 32 * gi
                poly, gl = g // gpp, g % gpp
                hi = gl // lo
                out.append(poly * n + hi * (n >> s) + gl % lo + i * lo)
            yield out


def wavefronts(addrs, phys) -> int:
    w = 0
    for half in (addrs[:16], addrs[16:]):
        banks: dict[int, set[int]] = {}
        for a in half:
            banks.setdefault(phys(a) % 16, set()).add(phys(a))
        w += max(len(v) for v in banks.values())
    return w


def schedules():
    for logn in range(4, 11):
        yield logn, 32          # k_warp LZ split-tail schedule
        yield logn, 3           # k_warp [0, 4q) radix-8 schedule
    yield 8, 3                  # k_rows (n2 = 8)


def total(phys):
    got = ideal = 0
    for logn, km in schedules():
        for s, k in passes(logn, km):
            for a in accesses(logn, s, k):
                got += wavefronts(a, phys)
                ideal += 2
    return got, ideal


if __name__ == "__main__":
    for name, f in (("swizzle", wswz), ("pad j + j>>4 (round 1)", pad)):
        got, ideal = total(f)
        print(f"{name}: {got} wavefronts, ideal {ideal} ({got / ideal:.3f}x)")
