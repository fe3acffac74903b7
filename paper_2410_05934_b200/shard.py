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


def efficiency(parts: list[Part], world: int) -> float:
    """Ideal parallel efficiency of the split: mean shard weight / max."""
    sh = plan(parts, world)
    ws = [shard_weight(parts, s) for s in sh]
    return (sum(ws) / world) / max(ws)
