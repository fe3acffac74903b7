"""Benchmark: batched negacyclic NTT -> (.) -> INTT on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg5]
                    [--impl ours|reference] [--scaling weak|strong]

One *step* is one pass of the whole hot path
over one batch of synthetic input: for every (polynomial, limb) unit,
c = INTT(NTT(a) (.) b_hat) (Eq. 1; reading C8: b_hat is an
NTT-form operand resident on the device, like an evaluation key or an RGSW
row).  The default workload is BASELINE.json configs[4] (cfg5), the config
the metric names both halves of: N=2^16 x 45 limbs (CKKS) plus N=2^10 x 16384
polynomials (TFHE).  `value` counts limb-transforms (one forward or one
inverse N-point transform of one limb) per second over all ranks.

Multi-GPU: `--gpus N` (N > 1) re-launches this script as N NCCL ranks
through torch.distributed.run unless it already runs under torchrun.  The
default for N > 1 is strong scaling: the fixed workload is split by limb and
polynomial with the weighted contiguous planner of SURVEY §8(e)
(paper_2410_05934_b200.shard); `--scaling weak` gives rank r polynomial block r
of a global problem of N copies.  Inputs are generated per shard from global
counters, so shards are slices of one global array; no collective touches the
data path.  After the timed region every rank digests its CUDA outputs per
unit, the digests are all-gathered and rank 0 compares their hash with the
oracle-computed hash in tests/golden/bench_digests.json (`digests_ok`).  With
`--scatter-gather` (N > 1) an `e2e_nccl` block times rank 0 scattering the
inputs over NCCL, the sharded compute, and the gather of the outputs to rank 0.
Timing: per-step CUDA events on the launching stream with an L2 flush
(>= 512 MiB write) between steps outside the events, W warm-up steps,
barrier + synchronize around the timed region, max over ranks.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import inputs  # noqa: E402

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
UNIT = "limb-transforms/s"

# Workloads (BASELINE.json configs).  parts: (log2n, limbs, polys, seed)
WORKLOADS = {
    "cfg1": {"desc": "N=2^10, one 60-bit prime, single polynomial, NTT -> (.) b_hat -> INTT",
             "parts": [(10, 1, 1, 0)]},
    "cfg2": {"desc": "N=2^10, one 60-bit prime, 4096 polynomials, NTT -> (.) b_hat -> INTT",
             "parts": [(10, 1, 4096, 0)]},
    "cfg3": {"desc": "N=2^16, 45 limbs, one polynomial, NTT -> (.) b_hat -> INTT",
             "parts": [(16, 45, 1, 0)]},
    "cfg4": {"desc": "N=2^16, 60 limbs x 8 polynomials, NTT -> (.) b_hat -> INTT",
             "parts": [(16, 60, 8, 0)]},
    "cfg5": {"desc": "N=2^16 x 45 limbs + N=2^10 x 16384 polynomials, NTT -> (.) b_hat -> INTT",
             "parts": [(16, 45, 1, 0), (10, 1, 16384, 0)]},
}

L2_FLUSH_BYTES = 512 << 20   # >= 4x the 126 MB L2 (SURVEY §8(d) timing protocol)
SPIN_CYCLES = 400_000   # ~200 us at 1.965 GHz: absorbs host jitter before the start event
FMA_SLOTS_PER_BFLY = 16   # exact Shoup butterfly: 6 wide/hi multiplies x 2 + 4 IMAD
IMAD_SLOTS_PER_CLK_SM = 64
N_SM = 148


def primes_for(logn: int, limbs: int):
    # Workload parameter, reading C2: the `limbs` largest primes q < 2^60 with
    # q = 1 mod 2N (the library validates them again in rnt_plan_create).
    two_n = 2 << logn
    out = []
    k = ((1 << 60) - 1) // two_n
    while len(out) < limbs:
        q = k * two_n + 1
        if _is_prime(q):
            out.append(q)
        k -= 1
    return out


def _is_prime(n: int) -> bool:
    if n < 2:
        return False
    for p in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int, period: float = 0.001):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None
        self.period = period

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            if self.period:
                time.sleep(self.period)

    def __enter__(self):
        if self._nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join()

    def summary(self):
        busy = [s for s in self.samples if s > 0]
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": self.max_mhz,
                "samples": len(self.samples), "reasons": sorted(self.reasons - {"gpu_idle"})}


# --------------------------------------------------------------- reference
def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def make_part_inputs(logn, limbs, polys, seed, poly_offset):
    mods = primes_for(logn, limbs)
    a = inputs.residues(seed, polys, mods, 1 << logn, batch_offset=poly_offset)
    bhat = inputs.residues(seed + 1, polys, mods, 1 << logn, batch_offset=poly_offset)
    return mods, a, bhat


def transforms_per_step(parts) -> int:
    return sum(2 * limbs * polys for (_, limbs, polys, _) in parts)


def bfly_per_step(parts) -> int:
    return sum(2 * limbs * polys * (1 << logn) // 2 * logn for (logn, limbs, polys, _) in parts)


def run_oracle_sample(parts, poly_offset: int, cores: int, min_seconds: float):
    """Time the CPU oracle (as it stands) on the workload; repeat until min_seconds."""
    import oracle as O

    data = []
    for (logn, limbs, polys, seed) in parts:
        mods, a, bhat = make_part_inputs(logn, limbs, polys, seed, poly_offset)
        psi = [O.min_psi(q, logn) for q in mods]
        data.append((mods, psi, a, bhat))
    reps, t0 = 0, time.perf_counter()
    while True:
        for mods, psi, a, bhat in data:
            O.batch(O.OP_POLYMUL_EVAL, a, mods, psi, b=bhat, n_threads=cores)
        reps += 1
        el = time.perf_counter() - t0
        if el >= min_seconds:
            break
    return reps, el


def cpu_baseline_block(wl, parts, cores, min_seconds=8.0, single_seconds=4.0):
    """The oracle as it stands on the host: all cores (the pthread pool over units)
    on the full workload, and one thread on a 1/64 sample."""
    reps, el = run_oracle_sample(parts, 0, cores, min_seconds)
    per = transforms_per_step(parts)
    small = reference_sample(parts, 64)
    reps1, el1 = run_oracle_sample(small, 0, 1, single_seconds)
    per1 = transforms_per_step(small)
    return {"value": per * reps / el, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
            "sample": f"full {wl} workload x {reps} repetition(s) ({per} limb-transforms each, "
                      f"{el:.1f} s wall on {cores} threads; oracle = plain C, exact 128-bit %)",
            "single_thread": {"value": per1 * reps1 / el1, "unit": UNIT, "cores": 1,
                              "sample": f"1/64 of {wl} ({per1} limb-transforms) x {reps1}, {el1:.1f} s on 1 thread"}}


def reference_sample(parts, frac: int = 8):
    """A bounded sample of the workload for the CPU reference arm: 1/frac of every
    part (limbs for the 2^16 part, polynomials for the batched part)."""
    out = []
    for (logn, limbs, polys, seed) in parts:
        if polys >= frac:
            out.append((logn, limbs, polys // frac, seed))
        else:
            out.append((logn, max(1, limbs // frac), polys, seed))
    return out


def bench_reference(args, wl, parts):
    import oracle as O

    ws, rank, _ = dist_env()
    if rank != 0:
        return
    cores = cpu_cores()
    sample = reference_sample(parts)
    per = transforms_per_step(sample)
    data = []
    for (logn, limbs, polys, seed) in sample:
        mods, a, bhat = make_part_inputs(logn, limbs, polys, seed, 0)
        data.append((mods, [O.min_psi(q, logn) for q in mods], a, bhat))

    def one_step():
        t0 = time.perf_counter()
        for mods, psi, a, bhat in data:
            O.batch(O.OP_POLYMUL_EVAL, a, mods, psi, b=bhat, n_threads=cores)
        return time.perf_counter() - t0

    for _ in range(args.warmup):
        one_step()
    times = [one_step() for _ in range(args.steps)]
    tot = sum(times)
    value = per * args.steps / tot
    desc = ", ".join(f"N=2^{lg} x {lm} limbs x {po} polys" for (lg, lm, po, _) in sample)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (seeded SplitMix64 uniform residues)",
        "config": {"workload": f"{wl}: {WORKLOADS[wl]['desc']}", "executor": "CPU oracle (plain C), all host cores",
                   "sample_per_step": desc},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"1/8 of {wl} per step ({desc}; {per} limb-transforms) on {cores} threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------ sharding + digests
GOLDEN_DIGESTS = os.path.join(ROOT, "tests", "golden", "bench_digests.json")


def plan_blocks(parts, ws: int, rank: int, scaling: str, planner: str = "contig"):
    """The blocks of the global job that `rank` owns.

    strong: the fixed workload is split by limb x polynomial with the weighted
    contiguous planner (paper_2410_05934_b200.shard, pure Python).  weak: rank r
    owns polynomial block r of a global problem of `ws` copies of the workload.
    A block is a dict: part index, log2n, the block's moduli, its global limb
    offset / total limbs, its polynomial count and global polynomial offset, seed.
    """
    from paper_2410_05934_b200 import shard as shd

    out = []
    if scaling == "weak":
        for pi, (logn, limbs, polys, seed) in enumerate(parts):
            out.append(dict(part=pi, logn=logn, mods=primes_for(logn, limbs), loff=0, ltot=limbs, polys=polys,
                            poff=rank * polys, seed=seed))
    else:
        sp = [shd.Part(lg, lm, po) for (lg, lm, po, _) in parts]
        for b in shd.PLANNERS[planner](sp, ws)[rank]:
            logn, limbs, polys, seed = parts[b.part]
            out.append(dict(part=b.part, logn=logn, mods=primes_for(logn, limbs)[b.limb_begin:b.limb_end],
                            loff=b.limb_begin, ltot=limbs, polys=b.poly_end - b.poly_begin, poff=b.poly_begin,
                            seed=seed))
    return out


def block_inputs(blk):
    """(a, b_hat) of a block: [polys][limbs][N] uint64 slices of the global arrays."""
    n = 1 << blk["logn"]
    a = inputs.residues_limbs(blk["seed"], blk["polys"], blk["mods"], n, blk["loff"], blk["ltot"],
                              batch_offset=blk["poff"])
    bh = inputs.residues_limbs(blk["seed"] + 1, blk["polys"], blk["mods"], n, blk["loff"], blk["ltot"],
                               batch_offset=blk["poff"])
    return a, bh


def block_digests(blk, c: np.ndarray):
    """Per-unit digest rows (part, global poly, global limb, sum, wsum) of a block's output."""
    rows = []
    for i in range(c.shape[0]):
        for j in range(c.shape[1]):
            s_, w_ = inputs.digest(c[i, j])
            rows.append((blk["part"], blk["poff"] + i, blk["loff"] + j, s_, w_))
    return rows


def gather_rows(rows, ws: int):
    """All-gather every rank's digest rows (any backend); every rank gets the union."""
    if ws == 1:
        return list(rows)
    import torch.distributed as dist

    got = [None] * ws
    dist.all_gather_object(got, list(rows))
    return [r for g in got for r in g]


def digests_sha(rows) -> str:
    arr = np.array(sorted(rows), dtype=np.uint64)
    return hashlib.sha256(arr.tobytes()).hexdigest()


def check_digests(wl: str, rows):
    """Compare the gathered digests with the oracle's (tests/golden, written by
    tools/make_golden_digests.py from oracle/ only).  None if no golden entry."""
    if not os.path.exists(GOLDEN_DIGESTS):
        return None
    g = json.load(open(GOLDEN_DIGESTS)).get(wl)
    if g is None:
        return None
    return len(rows) == g["units"] and digests_sha(rows) == g["sha256"]


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# --------------------------------------------------------------------- ours
def bench_ours(args, wl, parts):
    import torch

    import paper_2410_05934_b200 as R

    ws, rank, local = dist_env()
    # --emulate-rank R (testing): one process times rank R's shard of a --gpus N plan
    plan_ws, plan_rank = ws, rank
    if args.emulate_rank is not None:
        plan_ws, plan_rank = args.gpus, args.emulate_rank
    ndev = torch.cuda.device_count()
    # RNT_BENCH_SHARE_GPU=1 (testing the multi-rank path on a 1-GPU box only): ranks
    # share the visible GPUs and talk over gloo; never used for a reported number
    share = os.environ.get("RNT_BENCH_SHARE_GPU") == "1"
    if local >= ndev and not share:
        raise SystemExit(f"bench.py: local rank {local} but only {ndev} visible GPU(s)")
    local = local % ndev
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    backend = "gloo" if share else "nccl"
    red_dev = dev if backend == "nccl" else torch.device("cpu")
    if ws > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    stream = torch.cuda.current_stream()

    # ---- shard (plan_blocks): strong = the fixed workload split by limb x polynomial,
    # weak = rank r owns polynomial block r of ws copies
    blocks = plan_blocks(parts, plan_ws, plan_rank, args.scaling, args.shard)
    states = []
    for blk in blocks:
        a, bhat = block_inputs(blk)
        logn, mods = blk["logn"], blk["mods"]
        plan = R.Plan(logn, mods, device=local)
        da = torch.from_numpy(a.view(np.int64)).to(dev)
        db = torch.from_numpy(bhat.view(np.int64)).to(dev)
        dc = torch.empty_like(da)
        ha = torch.from_numpy(a.view(np.int64)).pin_memory()
        # two output / workspace sets: consecutive e2e steps alternate between them
        hc = [torch.empty_like(ha).pin_memory() for _ in range(2)]
        ws_buf = [torch.empty_like(da) for _ in range(2)]
        states.append(dict(logn=logn, limbs=len(mods), polys=blk["polys"], plan=plan, a=da, b=db, c=dc,
                           ha=ha, hc=hc, ws=ws_buf, blk=blk))
    # the dominant kernel: largest butterfly count part
    work = [(2 * s["limbs"] * s["polys"] * (1 << s["logn"]) // 2 * s["logn"]) for s in states]
    dom = int(np.argmax(work)) if work else 0
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)

    # independent parts (cfg5: the 2^16 x 45 polynomial and the 2^10 batch) run on
    # their own streams so each fills the other's ramp and tail (--sequential-parts: one stream)
    concurrent = args.concurrent_parts and len(states) > 1
    run_streams = [torch.cuda.Stream() for _ in states] if concurrent else [stream for _ in states]
    seq_streams = [stream for _ in states]

    def step(ev=None, span=None, streams=None, base=None):
        base = stream if base is None else base
        streams = run_streams if streams is None else streams
        if span is not None:
            span[0].record(base)
        order = list(enumerate(states))
        for i, s in (order[::-1] if args.reverse_parts else order):
            rs = streams[i]
            if rs is not base:
                rs.wait_stream(base)
            if ev is not None:
                ev[i][0].record(rs)
            R.polymul(s["plan"], s["c"], s["a"], s["b"], b_is_eval=True, stream=rs)
            if ev is not None:
                ev[i][1].record(rs)
        for rs in streams:
            if rs is not base:
                base.wait_stream(rs)
        if span is not None:
            span[1].record(base)

    # end to end: each part on its own user stream (independent batches overlap
    # their PCIe traffic); the library pipelines chunks inside each call.  Step k
    # uses buffer set / stream set k % 2, so step k+1's host->device copies queue
    # right behind step k's on the library's copy stream (streaming) while set k % 2
    # is reused only after step k - 2 completed (same user stream).
    part_streams = [[torch.cuda.Stream() for _ in states] for _ in range(2)]

    def step_host(k=0):
        sset = k % 2 if args.e2e_overlap else 0
        for s, ps in zip(states, part_streams[sset]):
            R.execute_host(s["plan"], R.OP_POLYMUL_EVAL, s["hc"][sset], s["ha"], s["ws"][sset], b_dev=s["b"],
                           stream=ps)

    def e2e_fork():
        ev = torch.cuda.Event()
        ev.record(stream)
        for pss in part_streams:
            for ps in pss:
                ps.wait_event(ev)

    def e2e_join():
        for pss in part_streams:
            for ps in pss:
                stream.wait_stream(ps)

    def barrier():
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()

    # ---- device-resident timed region
    evs = [[[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in states] for _ in range(args.steps)]
    spans = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    launches0 = R.launch_count()
    with ClockSampler(local) as clk:
        barrier()
        for k in range(args.steps):
            flush.zero_()   # L2 flush outside the timed events
            # device spin outside the events: the step's launches are queued before the
            # stream reaches the start event, so the events time device execution only
            torch.cuda._sleep(SPIN_CYCLES)
            step(evs[k], spans[k])
        barrier()
    launches = R.launch_count() - launches0
    part_ms = [[evs[k][i][0].elapsed_time(evs[k][i][1]) for k in range(args.steps)] for i in range(len(states))]
    step_ms = [spans[k][0].elapsed_time(spans[k][1]) for k in range(args.steps)]
    total_ms = sum(step_ms)

    # ---- per-kernel times for the roofline: with concurrent parts the timed
    # region overlaps them, so each part is also timed alone (one stream, L2
    # flushed, same spin) in a short sequential pass
    part_ms_seq = part_ms
    # collective on every rank (barriers inside) whenever the workload has several
    # parts -- a rank whose shard holds one part still takes part in the barriers
    if args.concurrent_parts and len(parts) > 1:
        nseq = min(args.steps, 20)
        sevs = [[[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in states] for _ in range(nseq)]
        barrier()
        for k in range(nseq):
            flush.zero_()
            torch.cuda._sleep(SPIN_CYCLES)
            step(sevs[k], None, seq_streams)
        barrier()
        part_ms_seq = [[sevs[k][i][0].elapsed_time(sevs[k][i][1]) for k in range(nseq)] for i in range(len(states))]

    # ---- secondary: L2-warm (no flush between steps; inputs partly L2-resident)
    warm_spans = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(min(args.steps, 50))]
    barrier()
    for sp in warm_spans:
        step(None, sp)
    barrier()
    warm_ms = statistics.mean(sp[0].elapsed_time(sp[1]) for sp in warm_spans)

    # ---- secondary: the step captured once in a CUDA graph and replayed (no host
    # launch work per step), L2 flushed between replays like the timed region
    graph = None
    if args.graph:
        # every rank takes part in the two barriers (a rank with an empty shard, or whose
        # capture failed, only waits), so the collectives stay matched across ranks
        g = None
        if states:
            try:
                g = torch.cuda.CUDAGraph()
                cap = torch.cuda.Stream()
                cap.wait_stream(stream)
                gstreams = [torch.cuda.Stream() for _ in states] if concurrent else [cap for _ in states]
                with torch.cuda.stream(cap):
                    with torch.cuda.graph(g, stream=cap):
                        step(None, None, gstreams, base=cap)
                stream.wait_stream(cap)
            except Exception as e:   # capture is an optional measurement; report why it is absent
                graph = {"error": f"{type(e).__name__}: {e}"[:200]}
                g = None
        gspans = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(min(args.steps, 50))]
        barrier()
        if g is not None:
            for sp in gspans:
                flush.zero_()
                torch.cuda._sleep(SPIN_CYCLES)
                sp[0].record(stream)
                g.replay()
                sp[1].record(stream)
        barrier()
        if g is not None:
            gms = [sp[0].elapsed_time(sp[1]) for sp in gspans]
            local_xf = sum(2 * st["limbs"] * st["polys"] for st in states)
            graph = {"ms_per_step": statistics.mean(gms), "median": statistics.median(gms),
                     "rank0_value": local_xf / (statistics.mean(gms) * 1e-3), "unit": UNIT,
                     "note": "secondary, rank 0: one step captured in a CUDA graph, replayed; L2 flushed"}
            del g

    # ---- end to end through the C ABI with host buffers (pinned), H2D + D2H inside
    e2e_ms = float("nan")
    if args.e2e:
        e2e_fork()
        for k in range(max(2, args.warmup // 2)):
            step_host(k)
        e2e_join()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record(stream)
        e2e_fork()
        for k in range(args.steps):
            if not args.e2e_overlap:
                e2e_join()
                e2e_fork()
            step_host(k)
        e2e_join()
        e1.record(stream)
        barrier()
        e2e_ms = e0.elapsed_time(e1)
    h2d = sum(s["a"].numel() * 8 for s in states)

    # ---- correctness of what was timed: per-unit digests of every rank's CUDA
    # outputs, all-gathered; rank 0 compares their hash with the oracle's
    # (tests/golden/bench_digests.json, written from oracle/ only)
    rows = []
    for st in states:
        rows += block_digests(st["blk"], st["c"].cpu().numpy().view(np.uint64))
    all_rows = gather_rows(rows, ws)
    digests_ok = (check_digests(wl, all_rows) if (args.scaling == "strong" or ws == 1) else None) \
        if args.emulate_rank is None else None
    e2e_match = None
    if args.e2e:   # the host-buffer path returned the same outputs as the device path
        last = (args.steps - 1) % 2 if args.e2e_overlap else 0
        e2e_match = all(torch.equal(st["hc"][last], st["c"].cpu()) for st in states)

    # ---- N > 1: end to end over NCCL (rank 0 scatters the inputs, gathers the outputs)
    nccl = None
    if ws > 1 and args.nccl_e2e and args.scaling == "strong" and backend == "nccl":
        nccl = scatter_gather_e2e(args, wl, parts, ws, rank, dev, stream, states, R, barrier)

    # distinct physical GPUs that ran a shard (device UUIDs gathered from every rank)
    try:
        my_gpu = str(torch.cuda.get_device_properties(dev).uuid)
    except Exception:
        my_gpu = f"{socket.gethostname()}:{local}"
    gpus_active = len(set(gather_rows([my_gpu], ws)))

    # ---- max over ranks
    t = torch.tensor([total_ms, e2e_ms], dtype=torch.float64, device=red_dev)
    if ws > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    total_ms, e2e_ms = float(t[0]), float(t[1])

    # units all ranks processed per step: weak = ws copies of the workload, strong = one
    global_xf = transforms_per_step(parts) * (ws if args.scaling == "weak" else 1)
    value = global_xf * args.steps / (total_ms * 1e-3)
    e2e_value = global_xf * args.steps / (e2e_ms * 1e-3)

    # ---- roofline of the dominant kernel(s)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    f_max = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    peak_bfly = N_SM * IMAD_SLOTS_PER_CLK_SM / FMA_SLOTS_PER_BFLY * f_max / 1e9   # Gbfly/s
    roof = None   # a rank with an empty shard (more ranks than units) only times and reports nothing
    if states:
        s = states[dom]
        bfly_launch = 2 * s["limbs"] * s["polys"] * (1 << s["logn"]) // 2 * s["logn"]
        dom_ms = statistics.mean(part_ms_seq[dom])   # rank 0's dominant kernel
        achieved = bfly_launch / (dom_ms * 1e-3) / 1e9
        traffic = None
        sass = None
        prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(prof):
            try:
                tj = json.load(open(prof))
                traffic = tj.get(f"{wl}:part{dom}")
                if states[dom]["logn"] == 10 and states[dom]["limbs"] * states[dom]["polys"] >= 3 * N_SM * 16:
                    sass = tj.get("sass:k_warp<10,2>")
            except Exception:
                traffic = None
        if s["limbs"] * s["polys"] <= 2:
            kern = f"k_clat / k_cluster <{s['logn']}> (single-launch cluster latency kernel)"
        elif s["logn"] <= 10:
            team = "4-warp" if s["logn"] == 10 and s["limbs"] * s["polys"] < 3 * N_SM * 16 else "2-warp"
            kern = (f"k_warp<{s['logn']},2> (fused NTT->(.)->INTT, one launch; lazy CT ranges, 3+3+2+2 passes, "
                    f"{team} teams, 32 warps/SM)")
        else:
            kern = f"k_col_fwd<{s['logn']}> + k_row<{s['logn']},2> + k_col_inv<{s['logn']}> (polymul, 3 launches)"
        # whole step: every butterfly of every part over the timed step time (all ranks)
        step_bfly = sum(2 * st["limbs"] * st["polys"] * (1 << st["logn"]) // 2 * st["logn"] for st in states) * (
            ws if args.scaling == "weak" else 1)
        step_achieved = step_bfly * args.steps / (total_ms * 1e-3) / 1e9 / ws
        # the polymul's other multiplies in butterfly equivalents (16 IMAD slots each): the
        # Montgomery (.) per coefficient (24 slots = 1.5) and the second Shoup product of the
        # last inverse stage's N/2 butterflies (N^-1 on both outputs, 1 each): 2N per unit
        pw_factor = 1.0 + 2.0 / s["logn"]
        roof = {"bound": "alu", "kernel": kern, "achieved": achieved, "peak": peak_bfly,
                "unit": "Gbutterfly/s", "frac": achieved / peak_bfly, "traffic": traffic,
                "frac_incl_pointwise": achieved * pw_factor / peak_bfly,
                "incl_pointwise_basis": f"x {pw_factor:.3f}: + 1.5 butterfly-equivalents per coefficient for the "
                                        "Montgomery (.) and + 1 per last-stage butterfly for the N^-1 product",
                "step_achieved_per_gpu": step_achieved, "step_frac": step_achieved / peak_bfly,
                "sass_per_butterfly": sass,
                "peak_basis": f"{N_SM} SMs x {IMAD_SLOTS_PER_CLK_SM} IMAD slots/clk / {FMA_SLOTS_PER_BFLY} slots "
                              f"per exact-Shoup butterfly x {f_max/1e6:.0f} MHz (sm_max_mhz)"}
    parts_out = []
    for i, st in enumerate(states):
        ms = statistics.mean(part_ms_seq[i])
        xf = 2 * st["limbs"] * st["polys"]
        bf = xf * (1 << st["logn"]) // 2 * st["logn"]
        alg_bytes = 3 * st["limbs"] * st["polys"] * (1 << st["logn"]) * 8  # read a, b_hat; write c
        parts_out.append({"log2n": st["logn"], "limbs": st["limbs"], "polys": st["polys"], "ms": ms,
                          "limb_transforms_per_s": xf / (ms * 1e-3),
                          "polynomials_per_s": st["polys"] / (ms * 1e-3),
                          "us_per_limb_transform": ms * 1e3 / xf,
                          "gbfly_per_s": bf / (ms * 1e-3) / 1e9, "frac_alu": bf / (ms * 1e-3) / 1e9 / peak_bfly,
                          "alg_hbm_gbs": alg_bytes / (ms * 1e-3) / 1e9})

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (seeded SplitMix64 uniform residues mod 60-bit NTT primes)",
            "config": {"workload": f"{wl}: {WORKLOADS[wl]['desc']}",
                       "l2": f"flushed ({L2_FLUSH_BYTES >> 20} MiB write) between steps, outside the timed events",
                       "launch": "a ~200 us device spin precedes each step's start event (outside the events): "
                                 "the events time device execution, not host launch latency",
                       "global_polys_per_part": [p[2] * (ws if args.scaling == 'weak' else 1) for p in parts],
                       "parallelism": (f"{'batch' if args.scaling == 'weak' else 'limb/batch'}-sharded x{ws} "
                                       f"({'N copies of the workload' if args.scaling == 'weak' else 'the fixed workload split by shard planner ' + args.shard}), "
                                       "no data-path collective")},
            "gpus_active": gpus_active,
            "process_group": backend if ws > 1 else None,
            "digests_ok": digests_ok,
            "digests": {"units": len(all_rows), "sha256": digests_sha(all_rows)[:16],
                        "against": "tests/golden/bench_digests.json (CPU oracle, tools/make_golden_digests.py)",
                        "e2e_outputs_equal_device_outputs": e2e_match},
            "gpu_launches": launches,
            "step_ms": {"mean": total_ms / args.steps, "median": statistics.median(step_ms), "min": min(step_ms),
                        "p90": sorted(step_ms)[int(0.9 * (len(step_ms) - 1))]},
            "l2_warm": {"ms_per_step": warm_ms,
                        "rank0_value": sum(2 * st["limbs"] * st["polys"] for st in states) / (warm_ms * 1e-3),
                        "note": "secondary: no L2 flush between steps, rank 0's shard"},
            "roofline": roof,
            "parts": parts_out,
            "parts_schedule": ("concurrent: the parts run on separate streams inside each timed step; roofline "
                               "and parts[].ms come from a sequential pass after the timed region (each part "
                               "alone, L2 flushed)") if concurrent else "sequential: one stream",
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": h2d,
                    "schedule": ("streamed: consecutive steps alternate two buffer sets, step k+1's copies queue "
                                 "behind step k's") if args.e2e_overlap else "serial: each step joins before the next"},
            "clocks": clk.summary(),
        }
        if graph is not None:
            line["cuda_graph"] = graph
        if nccl is not None:
            line["e2e_nccl"] = nccl
        if args.cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_block(wl, parts, cpu_cores())
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()



def scatter_gather_e2e(args, wl, parts, ws, rank, dev, stream, states, R, barrier):
    """N > 1, strong split: rank 0 holds the global inputs of every part on its GPU,
    scatters each rank's blocks over NCCL, every rank runs its polymuls, and the
    outputs are gathered back into rank 0's global arrays (NCCL only
    where a benchmark moves data).  Device time per step on each rank (CUDA events
    on the launching stream; the NCCL kernels are ordered against it), max over
    ranks by the caller's reduction below; rank 0 checks the gathered outputs'
    digests against the oracle's."""
    import torch
    import torch.distributed as dist

    layouts = [plan_blocks(parts, ws, r, "strong") for r in range(ws)]
    sizes = [sum(b["polys"] * len(b["mods"]) << b["logn"] for b in lay) for lay in layouts]
    mx = max(sizes)
    buf = torch.empty(mx, dtype=torch.int64, device=dev)
    glob = out = send = gath = None
    if rank == 0:
        glob = [torch.from_numpy(inputs.residues(seed, polys, primes_for(logn, limbs), 1 << logn).view(np.int64)).to(dev)
                for (logn, limbs, polys, seed) in parts]
        out = [torch.empty_like(g) for g in glob]
        send = [torch.empty(mx, dtype=torch.int64, device=dev) for _ in range(ws)]
        gath = [torch.empty(mx, dtype=torch.int64, device=dev) for _ in range(ws)]

    def slices(r, arrays, flat):
        off = 0
        for b in layouts[r]:
            g = arrays[b["part"]][b["poff"]:b["poff"] + b["polys"], b["loff"]:b["loff"] + len(b["mods"])]
            n = g.numel()
            yield g, flat[off:off + n].view(g.shape)
            off += n

    def one_step():
        if rank == 0:
            for r in range(ws):
                for g, f in slices(r, glob, send[r]):
                    f.copy_(g)
        dist.scatter(buf, send if rank == 0 else None, src=0)
        off = 0
        for st in states:
            n = st["a"].numel()
            st["a"].view(-1).copy_(buf[off:off + n])
            R.polymul(st["plan"], st["c"], st["a"], st["b"], b_is_eval=True, stream=stream)
            buf[off:off + n].copy_(st["c"].view(-1))
            off += n
        dist.gather(buf, gath if rank == 0 else None, dst=0)
        if rank == 0:
            for r in range(ws):
                for g, f in slices(r, out, gath[r]):
                    g.copy_(f)

    for _ in range(args.warmup):
        one_step()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        one_step()
    e1.record(stream)
    barrier()
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t[0])
    res = {"value": transforms_per_step(parts) / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms,
           "bytes_scattered_per_step": sum(sizes) * 8, "bytes_gathered_per_step": sum(sizes) * 8,
           "note": "rank 0's device-resident global inputs scattered over NCCL, sharded polymul, outputs "
                   "gathered to rank 0 (dist.scatter / dist.gather); device time, max over ranks"}
    if rank == 0:
        rows = []
        for pi, o in enumerate(out):
            h = o.cpu().numpy().view(np.uint64)
            blk = dict(part=pi, poff=0, loff=0)
            rows += block_digests(blk, h)
        res["digests_ok"] = check_digests(wl, rows)
    return res


# Paper-comparable single-polynomial latency: one 56-bit prime
# (P:616), one polynomial, forward NTT, N = 2^12 .. 2^16; quoted beside the
# paper's tab:ntt-mix A100 numbers (context only, other hardware).
PAPER_A100_M6_US = {12: 7.19, 13: 8.02, 14: 9.55, 15: 11.15, 16: 19.01}


def primes_below(bits: int, logn: int, count: int):
    two_n = 2 << logn
    k = ((1 << bits) - 1) // two_n
    out = []
    while len(out) < count:
        q = k * two_n + 1
        if _is_prime(q):
            out.append(q)
        k -= 1
    return out


def bench_latency(args):
    import torch

    import paper_2410_05934_b200 as R

    torch.cuda.set_device(0)
    res = {}
    for logn in range(12, 17):
        q = primes_below(56, logn, 1)
        plan = R.Plan(logn, q)
        a = inputs.residues(0, 1, q, 1 << logn)
        d = torch.from_numpy(a.view(np.int64)).cuda()
        o = torch.empty_like(d)
        for _ in range(20):
            R.ntt_forward(plan, o, d)
        torch.cuda.synchronize()
        # back-to-back (launch overhead overlapped) and isolated (synchronised) latency
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 200
        e0.record()
        for _ in range(reps):
            R.ntt_forward(plan, o, d)
        e1.record()
        torch.cuda.synchronize()
        b2b = e0.elapsed_time(e1) * 1e3 / reps
        iso = []
        for _ in range(50):
            e0.record()
            R.ntt_forward(plan, o, d)
            e1.record()
            torch.cuda.synchronize()
            iso.append(e0.elapsed_time(e1) * 1e3)
        # CUDA graph of 100 forward NTTs: GPU-side time per transform without Python launch overhead
        g = torch.cuda.CUDAGraph()
        s_ = torch.cuda.Stream()
        s_.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s_):
            R.ntt_forward(plan, o, d)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s_):
                for _ in range(100):
                    R.ntt_forward(plan, o, d)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(5):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        graph_us = e0.elapsed_time(e1) * 1e3 / 500
        res[f"2^{logn}"] = {"us_graph": graph_us, "us_back_to_back": b2b, "us_isolated_median": statistics.median(iso),
                            "paper_A100_M6_us": PAPER_A100_M6_US[logn], "q_bits": q[0].bit_length()}
    print(json.dumps({"mode": "latency", "metric": "single-polynomial forward NTT latency (us)",
                      "config": {"primes": "largest q < 2^56 with q = 1 mod 2N (P:616)", "polys": 1},
                      "results": res}), flush=True)


def bench_automorph(args):
    """NTT-domain Galois automorphism on cfg3/cfg4 shapes; memory-bound,
    roofline = HBM (16 B per element: read + write), L2 flushed between steps."""
    import torch

    import paper_2410_05934_b200 as R

    torch.cuda.set_device(0)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    res = {}
    for wl in ("cfg3", "cfg4"):
        (logn, limbs, polys, seed) = WORKLOADS[wl]["parts"][0]
        mods = primes_for(logn, limbs)
        plan = R.Plan(logn, mods)
        a = torch.from_numpy(inputs.residues(seed, polys, mods, 1 << logn).view(np.int64)).cuda()
        o = torch.empty_like(a)
        g = 5 ** 3 % (2 << logn)
        for _ in range(args.warmup):
            R.automorph(plan, o, a, g, ntt_domain=True)
        ms = []
        for _ in range(args.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            R.automorph(plan, o, a, g, ntt_domain=True)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        t = statistics.mean(ms)
        gbs = a.numel() * 16 / (t * 1e-3) / 1e9
        res[wl] = {"ms": t, "GBps": gbs, "frac_hbm": gbs / hbm}
    print(json.dumps({"mode": "automorph", "metric": "NTT-domain Galois automorphism HBM GB/s",
                      "roofline": {"bound": "hbm", "peak": hbm, "unit": "GB/s"}, "results": res}), flush=True)


def bench_extprod(args):
    """TFHE external product, n_slot ciphertexts (N=2^10, k=1) against one
    RGSW key (CMux-level batching), tab:tfhe parameters (1024, 630, 1, 3)
    -> l = 3 levels, base 2^20 (exact decomposition for the 60-bit prime)."""
    import torch

    import paper_2410_05934_b200 as R

    torch.cuda.set_device(0)
    logn, l, bg = 10, 3, 20
    n = 1 << logn
    res = {}
    mods = primes_for(logn, 1)
    plan = R.Plan(logn, mods)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    f_max = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    peak_bfly = N_SM * IMAD_SLOTS_PER_CLK_SM / FMA_SLOTS_PER_BFLY * f_max / 1e9
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    for n_slot in (1024, 4096, 16384):
        c = torch.from_numpy(inputs.residues(0, 2 * n_slot, mods, n).view(np.int64)).cuda()
        z = torch.from_numpy(inputs.residues(1, 2 * l * 2, mods, n).view(np.int64)).cuda()
        o = torch.empty_like(c)
        for _ in range(args.warmup):
            R.external_product(plan, o, c, z, bg, l, n_slot=n_slot)
        ms = []
        for _ in range(args.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            R.external_product(plan, o, c, z, bg, l, n_slot=n_slot)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        t = statistics.mean(ms)
        xf = n_slot * (2 * l + 2)
        bf = xf * (n // 2) * logn
        # the key MAC: 2 l x 2 Montgomery products per coefficient per slot (1.5 butterfly
        # equivalents each), and the inverses' last-stage second products (N/2 per transform)
        extra = n_slot * (4 * l * n * 1.5 + 2 * (n // 2))
        res[str(n_slot)] = {"ms": t, "external_products_per_s": n_slot / (t * 1e-3),
                            "limb_transforms_per_s": xf / (t * 1e-3),
                            "gbfly_per_s": bf / (t * 1e-3) / 1e9, "frac_alu": bf / (t * 1e-3) / 1e9 / peak_bfly,
                            "frac_alu_incl_mac": (bf + extra) / (t * 1e-3) / 1e9 / peak_bfly}
    # CPU oracle on a bounded sample
    import oracle as O

    cs = inputs.residues(0, 2 * 64, mods, n).reshape(64, 2, n)
    zs = inputs.residues(1, 2 * l * 2, mods, n).reshape(2 * l, 2, n)
    psi = O.min_psi(mods[0], logn)
    t0 = time.perf_counter()
    for sl in range(64):
        O.external_product(cs[sl], zs, mods[0], psi, bg, l)
    cpu = 64 / (time.perf_counter() - t0)
    print(json.dumps({"mode": "external_product", "metric": "TFHE external products/s (N=2^10, l=3, B=2^20)",
                      "roofline": {"bound": "alu", "peak": peak_bfly, "unit": "Gbutterfly/s"},
                      "results": res,
                      "cpu_baseline": {"value": cpu, "unit": "external products/s", "cores": 1, "kind": "oracle",
                                       "sample": "64 slots, single thread"}}), flush=True)


def bench_hrf(args):
    """HRF-MatVec of repack (tab:repack): out = add + sum_j pt_j (.) ct_j
    over n_slot precomputed rotation ciphertexts, NTT form, at N = 2^16 with 4 limbs (reading
    H2) and the paper's n_slot = 64 / 256 / 1024 (tab:sw).  HBM-bound: roofline = measured HBM
    bandwidth; algorithmic bytes = 24 n_slot L N (pt + both ct components read once) + 32 L N
    (add read, out written).  L2 flushed between steps (the inputs exceed L2 anyway)."""
    import torch

    import paper_2410_05934_b200 as R

    torch.cuda.set_device(0)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    logn, L = 16, 4
    n = 1 << logn
    mods = primes_for(logn, L)
    plan = R.Plan(logn, mods)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    res = {}
    for n_slot in (64, 256, 1024):
        pt = torch.from_numpy(inputs.residues(0, n_slot, mods, n).view(np.int64)).cuda()
        ct = torch.from_numpy(inputs.residues(1, 2 * n_slot, mods, n).view(np.int64)).cuda()
        add = torch.from_numpy(inputs.residues(2, 2, mods, n).view(np.int64)).cuda()
        out = torch.empty_like(add)
        for _ in range(args.warmup):
            R.hrf_matvec(plan, out, pt, ct, add=add)
        ms = []
        for _ in range(args.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            R.hrf_matvec(plan, out, pt, ct, add=add)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        t = statistics.mean(ms)
        alg = (24 * n_slot * L * n + 32 * L * n)
        gbs = alg / (t * 1e-3) / 1e9
        res[str(n_slot)] = {"ms": t, "ms_min": min(ms), "GBps": gbs, "frac_hbm": gbs / hbm,
                            "scalar_mults_per_s": 2 * n_slot * L * n / (t * 1e-3), "alg_bytes": alg}
        del pt, ct
        torch.cuda.empty_cache()
    # CPU oracle on a bounded sample: n_slot = 8, one limb
    import oracle as O

    pt = inputs.residues(0, 8, mods[:1], n)
    ct = inputs.residues(1, 16, mods[:1], n).reshape(8, 2, 1, n)
    t0 = time.perf_counter()
    reps = 0
    while time.perf_counter() - t0 < 3.0:
        O.hrf_matvec(pt, ct, mods[:1])
        reps += 1
    cpu = reps * 2 * 8 * n / (time.perf_counter() - t0)
    print(json.dumps({"mode": "hrf_matvec", "metric": "HRF-MatVec HBM GB/s (N=2^16, 4 limbs)",
                      "roofline": {"bound": "hbm", "peak": hbm, "unit": "GB/s"}, "results": res,
                      "cpu_baseline": {"value": cpu, "unit": "scalar modmults/s", "cores": 1, "kind": "oracle",
                                       "sample": "n_slot 8, one limb, N=2^16, single thread"}}), flush=True)


def bench_modup(args):
    """CKKS ModUp of one key-switching digit at N=2^16 (dnum = 3 for L = 45:
    a 15-limb digit extended to the other 30 limbs + 15 special primes):
    INTT (15 limbs) -> BConv (15 -> 45) -> NTT (45 limbs); L2 flushed between steps."""
    import torch

    import paper_2410_05934_b200 as R

    torch.cuda.set_device(0)
    logn, Lin, Kout = 16, 15, 45
    mods = primes_for(logn, Lin + Kout)
    src, dst = mods[:Lin], mods[Lin:]
    ps, pd = R.Plan(logn, src), R.Plan(logn, dst)
    bc = R.BConv(ps, pd)
    a = torch.from_numpy(inputs.residues(0, 1, src, 1 << logn).view(np.int64)).cuda()
    coeff = torch.empty_like(a)
    ext = torch.empty((1, Kout, 1 << logn), dtype=torch.int64, device="cuda")
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device="cuda")

    def step(ev):
        ev[0].record()
        R.ntt_inverse(ps, coeff, a)
        ev[1].record()
        bc(ext, coeff)
        ev[2].record()
        R.ntt_forward(pd, ext, ext)
        ev[3].record()

    for _ in range(args.warmup):
        step([torch.cuda.Event(enable_timing=True) for _ in range(4)])
    parts = [[], [], []]
    for _ in range(args.steps):
        flush.zero_()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        step(ev)
        torch.cuda.synchronize()
        for k in range(3):
            parts[k].append(ev[k].elapsed_time(ev[k + 1]))
    ms = [statistics.mean(x) for x in parts]
    n = 1 << logn
    print(json.dumps({"mode": "modup", "metric": "CKKS ModUp of one digit (INTT -> BConv -> NTT), N=2^16",
                      "config": {"digit_limbs": Lin, "target_limbs": Kout},
                      "ms": {"intt": ms[0], "bconv": ms[1], "ntt": ms[2], "total": sum(ms)},
                      "bconv_modmul_per_s": n * Lin * (Kout + 1) / (ms[1] * 1e-3),
                      "limb_transforms_per_s": (Lin + Kout) / (ms[0] * 1e-3 + ms[2] * 1e-3)}), flush=True)


def bench_keyswitch(args):
    """CKKS hybrid key switching (rnt_keyswitch_apply) and HROT =
    automorph(c0), automorph(c1), key switch of sigma(c1) with sigma(c0) added,
    at the paper's (N, L, dnum) = (2^16, 44 + 1 = 45 limbs, 45) with one
    special prime (reading KS1), and a dnum = 3 hybrid variant (15 special primes).
    Context, not a target: the paper's HEROT on A100 is 5.13 ms (tab:ckks-gpu-performance)."""
    import torch

    import paper_2410_05934_b200 as R

    torch.cuda.set_device(0)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    f_max = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    peak_bfly = N_SM * IMAD_SLOTS_PER_CLK_SM / FMA_SLOTS_PER_BFLY * f_max / 1e9
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    res = {}
    logn = 16
    n = 1 << logn
    for (L, K, dnum) in ((45, 1, 45), (45, 15, 3)):
        mods = primes_for(logn, L + K)
        qs = mods[:L]
        qp, qpp = R.Plan(logn, qs), R.Plan(logn, mods)
        ks = R.KeySwitch(qp, qpp, dnum)
        c = torch.from_numpy(inputs.residues(0, 2, qs, n).view(np.int64)).cuda()          # ciphertext (c0, c1)
        evk = torch.from_numpy(inputs.residues(1, 2 * dnum, mods, n).view(np.int64)).cuda()
        sc = torch.empty_like(c)
        out = torch.empty_like(c)
        g = 5                                                                            # rotation by one slot
        per = L * n

        def hrot():
            R.automorph(qp, sc, c, g, ntt_domain=True)
            ks(out, sc[1], evk, add0=sc[0])

        def kswitch():
            ks(out, c[1], evk)

        for name, fn in (("keyswitch", kswitch), ("hrot", hrot)):
            for _ in range(args.warmup):
                fn()
            ms = []
            for _ in range(args.steps):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                torch.cuda.synchronize()
                ms.append(e0.elapsed_time(e1))
            t = statistics.mean(ms)
            xf = L + dnum * (L + K) + 2 * K + 2 * L
            bf = xf * (n // 2) * logn
            res[f"L{L}_K{K}_dnum{dnum}_{name}"] = {
                "ms": t, "ms_min": min(ms), "ms_p90": sorted(ms)[int(0.9 * (len(ms) - 1))],
                "limb_transforms": xf, "gbfly_per_s": bf / (t * 1e-3) / 1e9,
                "frac_alu_transforms_only": bf / (t * 1e-3) / 1e9 / peak_bfly,
                "evk_GB": evk.numel() * 8 / 1e9,
                "evk_read_floor_ms": evk.numel() * 8 / (hbm * 1e9) * 1e3}
        del ks, evk
        torch.cuda.empty_cache()
    print(json.dumps({"mode": "keyswitch", "metric": "CKKS hybrid key switch / HROT latency (ms), N=2^16",
                      "paper_context": {"HEROT_ms_A100_Chameleon": 5.13, "params": "(2^16, logQ 2305, L 44, dnum 45)",
                                        "cite": "PAPER.md tab:ckks-gpu-performance (P:849-856)"},
                      "roofline": {"bound": "alu", "peak": peak_bfly, "unit": "Gbutterfly/s"},
                      "results": res}), flush=True)


def free_port() -> int:
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    return port


def relaunch_cmd(n: int, argv) -> list:
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
            "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *argv]


def relaunch(n: int, argv) -> int:
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.call(relaunch_cmd(n, argv), env=env)


def launch_check(args):
    """The multi-rank plumbing of bench_ours without a GPU: gloo process group,
    shard plan, per-shard input generation, digest all-gather, max-over-ranks
    reduction.  Digests are of the generated INPUTS (no method arithmetic), and
    rank 0 compares them with those of the unsharded inputs."""
    import torch
    import torch.distributed as dist

    ws, rank, _ = dist_env()
    if ws > 1:
        dist.init_process_group("gloo")
    parts = WORKLOADS[args.workload]["parts"]
    rows = []
    for blk in plan_blocks(parts, ws, rank, args.scaling, args.shard):
        a, _ = block_inputs(blk)
        rows += block_digests(blk, a)
    all_rows = gather_rows(rows, ws)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        want = []
        glob_ws = ws if args.scaling == "weak" else 1
        for pi, (logn, limbs, polys, seed) in enumerate(parts):
            blk = dict(part=pi, logn=logn, mods=primes_for(logn, limbs), loff=0, ltot=limbs,
                       polys=polys * glob_ws, poff=0, seed=seed)
            want += block_digests(blk, block_inputs(blk)[0])
        print(json.dumps({"launch_check": True, "n_gpus": ws, "scaling": args.scaling, "units": len(all_rows),
                          "digests_match": digests_sha(all_rows) == digests_sha(want), "max_rank": float(t[0])}),
              flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="cfg5", choices=sorted(WORKLOADS))
    ap.add_argument("--log2n", type=int, default=None,
                    help="custom workload instead of a preset: N = 2^log2n (with --limbs, --batch, --seed)")
    ap.add_argument("--limbs", type=int, default=1)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default=None, choices=["weak", "strong"],
                    help="strong (default): the fixed workload split over the ranks; weak: N copies")
    ap.add_argument("--scatter-gather", dest="nccl_e2e", action="store_true",
                    help="N > 1: add an e2e_nccl block (rank 0 scatters the inputs over NCCL, gathers the outputs)")
    ap.add_argument("--no-graph", dest="graph", action="store_false", help="skip the CUDA-graph replay block")
    ap.add_argument("--launch-check", action="store_true",
                    help="(tests) run the multi-rank launcher, shard plan and digest gather on CPU/gloo; "
                         "digests of the generated inputs, no compute")
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--no-e2e", dest="e2e", action="store_false", help="skip the host-buffer phase (profiling)")
    ap.add_argument("--e2e-serial", dest="e2e_overlap", action="store_false",
                    help="e2e: join every step before the next (default: consecutive steps stream)")
    ap.add_argument("--shard", default="parts", choices=["contig", "mixed", "parts"],
                    help="strong-scaling shard planner (shard.py): whole ranks per part when world >= 2 x parts, "
                         "else the contiguous weighted split (parts, default); contig; every rank a slice of "
                         "every part (mixed)")
    ap.add_argument("--emulate-rank", type=int, default=None,
                    help="testing: one process times rank R's shard of the --gpus N plan (no process group)")
    ap.add_argument("--reverse-parts", action="store_true",
                    help="launch the parts of a step in reverse order (experiment: cfg5 k_warp first)")
    ap.add_argument("--sequential-parts", dest="concurrent_parts", action="store_false",
                    help="run the parts of a step one after another on one stream (default: concurrent)")
    ap.add_argument("--concurrent-parts", dest="concurrent_parts", action="store_true",
                    help="run the independent parts of a step on separate streams")
    ap.add_argument("--latency", action="store_true", help="paper-comparable single-polynomial latency mode")
    ap.add_argument("--automorph", action="store_true", help="SURVEY f4 automorph bandwidth mode")
    ap.add_argument("--extprod", action="store_true", help="SURVEY f1 TFHE external product mode")
    ap.add_argument("--modup", action="store_true", help="SURVEY f2 CKKS ModUp (INTT -> BConv -> NTT) mode")
    ap.add_argument("--keyswitch", action="store_true", help="SURVEY f2 CKKS key switch / HROT mode")
    ap.add_argument("--hrf", action="store_true", help="SURVEY f4 HRF-MatVec scalar multiply-accumulate mode")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.scaling is None:
        args.scaling = "strong"
    single = args.latency or args.automorph or args.extprod or args.modup or args.keyswitch or args.hrf
    if (args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours" and not single
            and args.emulate_rank is None):
        # one process per GPU: re-launch this script under torch.distributed.run
        sys.exit(relaunch(args.gpus, sys.argv[1:]))
    if args.log2n is not None:
        # a custom single-part workload (reading-C2 primes); no golden digests (digests_ok: null)
        WORKLOADS["custom"] = {"desc": f"N=2^{args.log2n}, {args.limbs} limbs x {args.batch} polynomials, "
                                       f"seed {args.seed}, NTT -> (.) b_hat -> INTT",
                               "parts": [(args.log2n, args.limbs, args.batch, args.seed)]}
        args.workload = "custom"
    if args.launch_check:
        return launch_check(args)
    wl = args.workload
    parts = WORKLOADS[wl]["parts"]
    if args.latency:
        bench_latency(args)
    elif args.automorph:
        bench_automorph(args)
    elif args.extprod:
        bench_extprod(args)
    elif args.modup:
        bench_modup(args)
    elif args.keyswitch:
        bench_keyswitch(args)
    elif args.hrf:
        bench_hrf(args)
    elif args.impl == "reference":
        bench_reference(args, wl, parts)
    else:
        bench_ours(args, wl, parts)


if __name__ == "__main__":
    main()
