"""Limb x batch shard planner for multi-GPU runs.

Every (polynomial b, limb l) unit of every part is an independent transform
(RNS limbs are independent; polynomials of a batch are independent,
P:324-332), so a job shards with no data-path collective.  Units are ordered
part-major, then limb-major, then polynomial; each unit weighs its butterfly
count (N/2) log2 N, so a 2^16 limb weighs 102.4 of a 2^10 polynomial.  Rank r
receives the contiguous unit range whose cumulative weight falls in
[r W / world, (r+1) W / world).

A shard is a list of Blocks (part, limb range, polynomial range); a block
always covers a rectangle, so it maps onto one plan (for its limbs' primes)
and one [polys][limbs][N] array.  Pure Python, no device code.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Part:
    log2n: int
    limbs: int
    polys: int

    @property
    def weight(self) -> int:  # butterflies per (poly, limb) unit
        return (1 << self.log2n) // 2 * self.log2n


@dataclass(frozen=True)
class Block:
    part: int
    limb_begin: int
    limb_end: int
    poly_begin: int
    poly_end: int

    @property
    def units(self) -> int:
        return (self.limb_end - self.limb_begin) * (self.poly_end - self.poly_begin)


def _cut_points(parts, world):
    total = sum(p.weight * p.limbs * p.polys for p in parts)
    return [total * r // world for r in range(world + 1)], total


def plan(parts: list[Part], world: int) -> list[list[Block]]:
    """Contiguous weighted split of all units into `world` shards."""
    if world < 1:
        raise ValueError("world >= 1")
    cuts, _ = _cut_points(parts, world)
    shards: list[list[Block]] = [[] for _ in range(world)]
    acc = 0  # cumulative weight before the current unit
    for pi, p in enumerate(parts):
        for l in range(p.limbs):
            # units (l, b) for b in [0, polys): weights acc + b*w
            b = 0
            while b < p.polys:
                start = acc + b * p.weight
                # rank owning this unit: largest r with cuts[r] <= start (by unit start weight)
                r = max(i for i in range(world) if cuts[i] <= start)
                # how many consecutive polys stay in rank r
                end_w = cuts[r + 1]
                nb = max(1, min(p.polys - b, -(-(end_w - start) // p.weight)))
                shards[r].append(Block(pi, l, l + 1, b, b + nb))
                b += nb
            acc += p.polys * p.weight
    return [_merge(s) for s in shards]


def plan_mixed(parts: list[Part], world: int) -> list[list[Block]]:
    """Every rank gets a slice of every part (cfg5: ~45/world limbs of the 2^16
    polynomial and ~16384/world of the 2^10 batch), so each rank runs the same mix
    as one GPU does and its parts overlap on two streams.  The parts with coarse
    units are split evenly by unit count (a rank's share differs by at most one
    unit); the part with the finest units then fills every rank up to the mean
    weight, which evens out the coarse parts' rounding."""
    if world < 1:
        raise ValueError("world >= 1")
    shards: list[list[Block]] = [[] for _ in range(world)]
    load = [0] * world
    order = sorted(range(len(parts)), key=lambda i: -parts[i].weight)
    fine = order[-1]

    def units_to_blocks(pi, u0, u1):
        """Units [u0, u1) of part pi (limb-major: unit = l * polys + b) as rectangles."""
        p = parts[pi]
        out = []
        u = u0
        while u < u1:
            l, b = divmod(u, p.polys)
            nb = min(p.polys - b, u1 - u)
            out.append(Block(pi, l, l + 1, b, b + nb))
            u += nb
        return out

    for pi in order[:-1]:
        p = parts[pi]
        n = p.limbs * p.polys
        for r in range(world):
            u0, u1 = n * r // world, n * (r + 1) // world
            shards[r] += units_to_blocks(pi, u0, u1)
            load[r] += (u1 - u0) * p.weight
    p = parts[fine]
    n = p.limbs * p.polys
    total = sum(load) + n * p.weight
    u = 0
    for r in range(world):
        # fine units for rank r: fill up to the cumulative target (last rank takes the rest)
        target = total * (r + 1) // world - sum(load[: r + 1]) - u * p.weight
        k = n - u if r == world - 1 else max(0, min(n - u, round(target / p.weight)))
        shards[r] += units_to_blocks(fine, u, u + k)
        u += k
    return [_merge(s) for s in shards]


def plan_by_part(parts: list[Part], world: int) -> list[list[Block]]:
    """Whole ranks per part: part p gets k_p ranks, k_p proportional to its weight
    (largest remainder, at least one each), and its units are split contiguously
    among them -- so no rank runs two kernel chains and pays both parts' fixed
    costs (launch ramps and tails dominate a rank's step at 8 GPUs: one 2^16 x 45
    chain costs ~36 us before its first limb, the 2^10 batch ~18 us).  Needs
    world >= 2 x parts, else the contiguous split (plan)."""
    if world < 2 * len(parts):
        return plan(parts, world)
    w = [p.weight * p.limbs * p.polys for p in parts]
    total = sum(w)
    k = [max(1, int(world * x // total)) for x in w]
    while sum(k) < world:   # largest remainder
        i = max(range(len(parts)), key=lambda j: world * w[j] / total - k[j])
        k[i] += 1
    while sum(k) > world:
        i = max(range(len(parts)), key=lambda j: k[j] - world * w[j] / total if k[j] > 1 else -1e9)
        k[i] -= 1
    shards: list[list[Block]] = []
    for pi, p in enumerate(parts):
        sub = plan([p], k[pi])
        for sh in sub:
            shards.append([Block(pi, b.limb_begin, b.limb_end, b.poly_begin, b.poly_end) for b in sh])
    return shards


PLANNERS = {"contig": plan, "mixed": plan_mixed, "parts": plan_by_part}


def _merge(blocks: list[Block]) -> list[Block]:
    """Merge consecutive single-limb blocks with identical poly ranges."""
    out: list[Block] = []
    for bl in blocks:
        if out:
            last = out[-1]
            if (last.part == bl.part and last.limb_end == bl.limb_begin and last.poly_begin == bl.poly_begin
                    and last.poly_end == bl.poly_end):
                out[-1] = Block(last.part, last.limb_begin, bl.limb_end, last.poly_begin, last.poly_end)
                continue
        out.append(bl)
    return out


def shard_weight(parts: list[Part], shard: list[Block]) -> int:
    return sum(parts[b.part].weight * b.units for b in shard)


def efficiency(parts: list[Part], world: int, planner: str = "contig") -> float:
    """Ideal parallel efficiency of the split: mean shard weight / max."""
    sh = PLANNERS[planner](parts, world)
    ws = [shard_weight(parts, s) for s in sh]
    return (sum(ws) / world) / max(ws)
