"""Multi-process (world_size 2, gloo, CPU) tests of the sharded orchestration:
the limb x batch shard planner, shard-local input
generation from global counters, and digest gathering.  Each rank computes
its shard with the CPU oracle; rank 0 checks the gathered per-unit digests
against the unsharded computation.  The bench.py launcher itself (`--gpus 2`
re-launching under torch.distributed.run) and its shard / digest helpers are
driven here on CPU too.  No GPU needed."""
import importlib.util
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _shard_module():
    spec = importlib.util.spec_from_file_location("rnt_shard", os.path.join(ROOT, "paper_2410_05934_b200", "shard.py"))
    m = importlib.util.module_from_spec(spec)
    sys.modules["rnt_shard"] = m
    spec.loader.exec_module(m)
    return m


S = _shard_module()
PARTS = [S.Part(10, 3, 5), S.Part(12, 2, 3), S.Part(5, 1, 40)]


def _primes(logn, limbs):
    import oracle as O

    return O.primes(logn, limbs)


def _unit_digests(parts, blocks, seed_base=0):
    """Oracle polymul-eval on each block; digest per (part, poly, limb)."""
    import inputs
    import oracle as O

    out = {}
    for b in blocks:
        p = parts[b.part]
        mods_all = _primes(p.log2n, p.limbs)
        mods = mods_all[b.limb_begin:b.limb_end]
        psi = [O.min_psi(q, p.log2n) for q in mods]
        n = 1 << p.log2n
        seed = seed_base + 10 * b.part
        a = inputs.residues_limbs(seed, b.poly_end - b.poly_begin, mods, n, b.limb_begin, p.limbs,
                                  batch_offset=b.poly_begin)
        bh = inputs.residues_limbs(seed + 1, b.poly_end - b.poly_begin, mods, n, b.limb_begin, p.limbs,
                                   batch_offset=b.poly_begin)
        c = O.batch(O.OP_POLYMUL_EVAL, a, mods, psi, b=bh)
        for i in range(c.shape[0]):
            for j in range(c.shape[1]):
                out[(b.part, b.poly_begin + i, b.limb_begin + j)] = inputs.digest(c[i, j])
    return out


@pytest.mark.parametrize("planner", ["contig", "mixed", "parts"])
def test_plan_covers_every_unit_once(planner):
    for world in (1, 2, 3, 4, 5, 8):
        sh = S.PLANNERS[planner](PARTS, world)
        assert len(sh) == world
        seen = {}
        for r, blocks in enumerate(sh):
            for b in blocks:
                for l in range(b.limb_begin, b.limb_end):
                    for pb in range(b.poly_begin, b.poly_end):
                        key = (b.part, l, pb)
                        assert key not in seen
                        seen[key] = r
        want = {(pi, l, pb) for pi, p in enumerate(PARTS) for l in range(p.limbs) for pb in range(p.polys)}
        assert set(seen) == want


def test_plan_by_part_gives_whole_ranks_per_part():
    cfg5 = [S.Part(16, 45, 1), S.Part(10, 1, 16384)]
    sh = S.plan_by_part(cfg5, 8)
    parts_of = [{b.part for b in s} for s in sh]
    assert all(len(p) == 1 for p in parts_of)                      # no rank runs both chains
    assert [next(iter(p)) for p in parts_of].count(0) == 2          # 2 of 8 ranks take the 2^16 part
    assert sorted(sum(b.units for b in s) for s in sh[:2]) == [22, 23]
    assert S.plan_by_part(cfg5, 3) == S.plan(cfg5, 3)              # fewer than 2 ranks per part: contiguous
    assert S.plan_by_part([S.Part(10, 1, 4096)], 8) == S.plan([S.Part(10, 1, 4096)], 8)


def test_plan_balance_matches_survey_table():
    # SURVEY §8(e) ideal efficiencies
    cfg3 = [S.Part(16, 45, 1)]
    assert abs(S.efficiency(cfg3, 2) - 0.978) < 1e-3
    assert abs(S.efficiency(cfg3, 8) - 0.9375) < 1e-4
    assert S.efficiency([S.Part(16, 60, 8)], 8) == 1.0
    assert S.efficiency([S.Part(10, 1, 4096)], 8) == 1.0
    assert S.efficiency([S.Part(16, 45, 1), S.Part(10, 1, 16384)], 8) > 0.98


def test_shard_inputs_are_slices_of_global_inputs():
    import inputs

    mods = _primes(10, 3)
    full = inputs.residues(4, 6, mods, 1024)
    part = inputs.residues_limbs(4, 2, mods[1:3], 1024, 1, 3, batch_offset=3)
    assert np.array_equal(part, full[3:5, 1:3])
    assert np.array_equal(inputs.residues(4, 2, mods, 1024, batch_offset=4), full[4:6])


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shard = _shard_module()
        parts = [shard.Part(10, 3, 5), shard.Part(12, 2, 3), shard.Part(5, 1, 40)]
        mine = _unit_digests(parts, shard.plan(parts, world)[rank])
        gathered = [None] * world
        dist.all_gather_object(gathered, mine)
        # max-over-ranks timing reduction used by bench.py
        import torch

        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            merged = {}
            for g in gathered:
                assert not (set(merged) & set(g))
                merged.update(g)
            full = _unit_digests(parts, [shard.Block(i, 0, p.limbs, 0, p.polys) for i, p in enumerate(parts)])
            q.put((merged == full, len(merged), float(t[0])))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.timeout(300)
def test_gloo_world2_sharded_digests_equal_unsharded():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
        assert p.exitcode == 0
    ok, n, tmax = q.get(timeout=10)
    assert ok and n == sum(p.limbs * p.polys for p in PARTS)
    assert tmax == 2.0


def _bench_module():
    spec = importlib.util.spec_from_file_location("rnt_bench", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    sys.modules["rnt_bench"] = m
    spec.loader.exec_module(m)
    return m


def _bench_worker(rank, world, port, wl, q):
    """bench.py's own shard plan / input / digest / gather helpers, the CUDA compute
    replaced by the oracle (test infrastructure): the gathered hash must equal the
    golden oracle hash bench.py checks on the GPU (tests/golden/bench_digests.json)."""
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O

        B = _bench_module()
        parts = B.WORKLOADS[wl]["parts"]
        rows = []
        for blk in B.plan_blocks(parts, world, rank, "strong"):
            a, bh = B.block_inputs(blk)
            psi = [O.min_psi(qq, blk["logn"]) for qq in blk["mods"]]
            c = O.batch(O.OP_POLYMUL_EVAL, a, blk["mods"], psi, b=bh, n_threads=4)
            rows += B.block_digests(blk, c)
        allr = B.gather_rows(rows, world)
        if rank == 0:
            q.put((B.check_digests(wl, allr), len(allr), len(rows)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("wl", ["cfg3", "cfg2"])
def test_gloo_world2_bench_shards_match_golden_digests(wl):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, 2, port, wl, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(280)
        assert p.exitcode == 0
    ok, n, n0 = q.get(timeout=10)
    assert ok is True
    assert 0 < n0 < n   # rank 0 owned a strict part of the units


def test_bench_relaunch_command():
    B = _bench_module()
    cmd = B.relaunch_cmd(8, ["--gpus", "8", "--steps", "3"])
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=8" in cmd and "127.0.0.1" in cmd
    assert cmd[-3:] == ["--gpus", "8", "--steps", "3"][-3:] and cmd[-4] == "--gpus"


@pytest.mark.timeout(300)
def test_bench_gpus4_launcher_gloo_parts_planner():
    """`bench.py --gpus 4` (strong, default planner: whole ranks per part) over gloo:
    every unit of cfg5 planned exactly once and the gathered digests match."""
    import json
    import subprocess

    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--launch-check",
                        "--workload", "cfg5"], capture_output=True, text=True, timeout=280, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][0])
    assert d["n_gpus"] == 4 and d["digests_match"] is True and d["units"] == 45 + 16384


@pytest.mark.timeout(300)
@pytest.mark.parametrize("scaling", ["strong", "weak"])
def test_bench_gpus2_launcher_gloo(scaling):
    """`bench.py --gpus 2` without torchrun env re-launches itself as 2 ranks; the
    ranks plan their shards, generate their inputs and all-gather digests."""
    import json
    import subprocess

    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--launch-check",
                        "--workload", "cfg5", "--scaling", scaling], capture_output=True, text=True, timeout=280,
                       cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["digests_match"] is True and d["max_rank"] == 2.0
    assert d["units"] == (45 + 16384) * (2 if scaling == "weak" else 1)
