"""Write tests/golden/bench_digests.json: the per-unit output digests of every
bench workload (BASELINE.json configs, bench.py WORKLOADS) computed by the CPU
oracle alone.

    python tools/make_golden_digests.py [cfg1 cfg2 ...]

A step of the bench computes, for every (polynomial b, limb l) unit of every
part, c = INTT(NTT(a) (.) b_hat) (Eq. 1; reading C8: b_hat is the
seed + 1 residue array taken as an NTT-form operand).  The digest of a unit is
inputs.digest(c[b][l]) = (sum c_i, sum (i+1) c_i) mod 2^64.
Rows (part, poly, limb, sum, wsum) are sorted and hashed with SHA-256; bench.py
all-gathers the digests of its CUDA outputs from every rank and compares the
hash (`digests_ok`).  Only oracle/ and inputs/ are called here (no product
code), so the stored values never come from the CUDA path.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import inputs  # noqa: E402
import oracle as O  # noqa: E402

# (log2n, limbs, polys, seed) per part -- the same shapes as bench.py WORKLOADS
WORKLOADS = {
    "cfg1": [(10, 1, 1, 0)],
    "cfg2": [(10, 1, 4096, 0)],
    "cfg3": [(16, 45, 1, 0)],
    "cfg4": [(16, 60, 8, 0)],
    "cfg5": [(16, 45, 1, 0), (10, 1, 16384, 0)],
}
OUT = os.path.join(ROOT, "tests", "golden", "bench_digests.json")


def digest_rows(parts, threads):
    rows = []
    for pi, (logn, limbs, polys, seed) in enumerate(parts):
        mods = O.primes(logn, limbs)          # reading C2
        psi = [O.min_psi(q, logn) for q in mods]   # reading C1
        n = 1 << logn
        chunk = max(1, 2048 // limbs)
        for p0 in range(0, polys, chunk):
            pc = min(chunk, polys - p0)
            a = inputs.residues(seed, pc, mods, n, batch_offset=p0)
            bh = inputs.residues(seed + 1, pc, mods, n, batch_offset=p0)
            c = O.batch(O.OP_POLYMUL_EVAL, a, mods, psi, b=bh, n_threads=threads)
            for i in range(pc):
                for l in range(limbs):
                    s, w = inputs.digest(c[i, l])
                    rows.append((pi, p0 + i, l, s, w))
    return rows


def sha(rows) -> str:
    arr = np.array(sorted(rows), dtype=np.uint64)
    return hashlib.sha256(arr.tobytes()).hexdigest()


def main():
    names = sys.argv[1:] or sorted(WORKLOADS)
    threads = len(os.sched_getaffinity(0))
    gold = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for wl in names:
        rows = digest_rows(WORKLOADS[wl], threads)
        gold[wl] = {"units": len(rows), "sha256": sha(rows),
                    "first": [list(map(int, r)) for r in sorted(rows)[:2]],
                    "parts": WORKLOADS[wl]}
        print(wl, gold[wl]["units"], gold[wl]["sha256"][:16], flush=True)
    gold["_source"] = ("tools/make_golden_digests.py: CPU oracle (oracle/ntt_oracle.c) on the seeded inputs of "
                       "inputs/; rows (part, poly, limb, sum, wsum) sorted, uint64, SHA-256")
    json.dump(gold, open(OUT, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
