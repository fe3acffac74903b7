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

Multi-GPU (torchrun): weak scaling by default -- rank r owns polynomial
batch index r of the global problem (inputs generated from the global
counters, so shards are slices of one global array); no collective touches
the data path.  Timing: per-step CUDA events on the launching stream with an
L2 flush (256 MiB write) between steps outside the events, W warm-up steps,
barrier + synchronize around the timed region, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
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

L2_FLUSH_BYTES = 256 << 20
SPIN_CYCLES = 100_000   # ~50 us at 1.965 GHz
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

    def __init__(self, index: int, period: float = 0.0):
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


def cpu_baseline_block(wl, parts, cores, min_seconds=8.0):
    reps, el = run_oracle_sample(parts, 0, cores, min_seconds)
    per = transforms_per_step(parts)
    return {"value": per * reps / el, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"full {wl} workload x {reps} repetition(s) ({per} limb-transforms each, "
                      f"{el:.1f} s wall on {cores} threads; oracle = plain C, exact 128-bit %)"}


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


# --------------------------------------------------------------------- ours
def bench_ours(args, wl, parts):
    import torch

    import paper_2410_05934_b200 as R

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream()

    # ---- shard.  weak: rank r owns global polynomial block r of every part.
    # strong: the fixed global job is split by limb x polynomial with the
    # weighted contiguous planner of SURVEY §8(e) (paper_2410_05934_b200.shard).
    from paper_2410_05934_b200 import shard as shd

    blocks = []   # (log2n, limbs_slice_mods, limb_offset, total_limbs, polys, poly_offset, seed)
    if args.scaling == "weak":
        for (logn, limbs, polys, seed) in parts:
            blocks.append((logn, primes_for(logn, limbs), 0, limbs, polys, rank * polys, seed))
    else:
        sp = [shd.Part(lg, lm, po) for (lg, lm, po, _) in parts]
        for b in shd.plan(sp, ws)[rank]:
            logn, limbs, polys, seed = parts[b.part]
            mods = primes_for(logn, limbs)[b.limb_begin:b.limb_end]
            blocks.append((logn, mods, b.limb_begin, limbs, b.poly_end - b.poly_begin, b.poly_begin, seed))
    states = []
    for (logn, mods, loff, ltot, polys, poff, seed) in blocks:
        a = inputs.residues_limbs(seed, polys, mods, 1 << logn, loff, ltot, batch_offset=poff)
        bhat = inputs.residues_limbs(seed + 1, polys, mods, 1 << logn, loff, ltot, batch_offset=poff)
        plan = R.Plan(logn, mods, device=local)
        da = torch.from_numpy(a.view(np.int64)).to(dev)
        db = torch.from_numpy(bhat.view(np.int64)).to(dev)
        dc = torch.empty_like(da)
        ha = torch.from_numpy(a.view(np.int64)).pin_memory()
        # two output / workspace sets: consecutive e2e steps alternate between them
        hc = [torch.empty_like(ha).pin_memory() for _ in range(2)]
        ws_buf = [torch.empty_like(da) for _ in range(2)]
        states.append(dict(logn=logn, limbs=len(mods), polys=polys, plan=plan, a=da, b=db, c=dc,
                           ha=ha, hc=hc, ws=ws_buf))
    # the dominant kernel: largest butterfly count part
    work = [(2 * s["limbs"] * s["polys"] * (1 << s["logn"]) // 2 * s["logn"]) for s in states]
    dom = int(np.argmax(work)) if work else 0
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)

    # independent parts (cfg5: the 2^16 x 45 polynomial and the 2^10 batch) run on
    # their own streams so each fills the other's ramp and tail (--sequential-parts: one stream)
    concurrent = args.concurrent_parts and len(states) > 1
    run_streams = [torch.cuda.Stream() for _ in states] if concurrent else [stream for _ in states]
    seq_streams = [stream for _ in states]

    def step(ev=None, span=None, streams=None):
        streams = run_streams if streams is None else streams
        if span is not None:
            span[0].record(stream)
        for i, s in enumerate(states):
            rs = streams[i]
            if rs is not stream:
                rs.wait_stream(stream)
            if ev is not None:
                ev[i][0].record(rs)
            R.polymul(s["plan"], s["c"], s["a"], s["b"], b_is_eval=True, stream=rs)
            if ev is not None:
                ev[i][1].record(rs)
        for rs in streams:
            if rs is not stream:
                stream.wait_stream(rs)
        if span is not None:
            span[1].record(stream)

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
    if concurrent:
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

    # ---- max over ranks
    t = torch.tensor([total_ms, e2e_ms], dtype=torch.float64, device=dev)
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
    s = states[dom]
    bfly_launch = 2 * s["limbs"] * s["polys"] * (1 << s["logn"]) // 2 * s["logn"]
    dom_ms = statistics.mean(part_ms_seq[dom])
    achieved = bfly_launch / (dom_ms * 1e-3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get(f"{wl}:part{dom}")
        except Exception:
            traffic = None
    kern = f"k_warp<{s['logn']},2> (fused NTT->(.)->INTT, one launch; lazy CT ranges, 3+3+2+2 passes)" \
        if s["logn"] <= 10 else \
        f"k_col_fwd<{s['logn']}> + k_row<{s['logn']},2> + k_col_inv<{s['logn']}> (polymul, 3 launches)"
    # whole step: every butterfly of every part over the timed step time (all ranks)
    step_bfly = sum(2 * st["limbs"] * st["polys"] * (1 << st["logn"]) // 2 * st["logn"] for st in states) * (
        ws if args.scaling == "weak" else 1)
    step_achieved = step_bfly * args.steps / (total_ms * 1e-3) / 1e9 / ws
    roof = {"bound": "alu", "kernel": kern, "achieved": achieved, "peak": peak_bfly,
            "unit": "Gbutterfly/s", "frac": achieved / peak_bfly, "traffic": traffic,
            "step_achieved_per_gpu": step_achieved, "step_frac": step_achieved / peak_bfly,
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
                       "l2": "flushed (256 MiB write) between steps, outside the timed events",
                       "launch": "a ~50 us device spin precedes each step's start event (outside the events): "
                                 "the events time device execution, not host launch latency",
                       "global_polys_per_part": [p[2] * (ws if args.scaling == 'weak' else 1) for p in parts],
                       "parallelism": f"{'batch' if args.scaling == 'weak' else 'limb/batch'}-sharded x{ws}, no data-path collective"},
            "gpu_launches": launches,
            "step_ms": {"mean": total_ms / args.steps, "median": statistics.median(step_ms), "min": min(step_ms),
                        "p90": sorted(step_ms)[int(0.9 * (len(step_ms) - 1))]},
            "l2_warm": {"ms_per_step": warm_ms, "value": transforms_per_step(parts) / (warm_ms * 1e-3),
                        "note": "secondary: no L2 flush between steps, rank 0"},
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
        if args.cpu_baseline and ws >= 1 and rank == 0 and (ws == 1):
            line["cpu_baseline"] = cpu_baseline_block(wl, parts, cpu_cores())
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()



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
        res[str(n_slot)] = {"ms": t, "external_products_per_s": n_slot / (t * 1e-3),
                            "limb_transforms_per_s": xf / (t * 1e-3),
                            "gbfly_per_s": bf / (t * 1e-3) / 1e9, "frac_alu": bf / (t * 1e-3) / 1e9 / peak_bfly}
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="cfg5", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--no-e2e", dest="e2e", action="store_false", help="skip the host-buffer phase (profiling)")
    ap.add_argument("--e2e-serial", dest="e2e_overlap", action="store_false",
                    help="e2e: join every step before the next (default: consecutive steps stream)")
    ap.add_argument("--sequential-parts", dest="concurrent_parts", action="store_false",
                    help="run the parts of a step one after another on one stream (default: concurrent)")
    ap.add_argument("--concurrent-parts", dest="concurrent_parts", action="store_true",
                    help="run the independent parts of a step on separate streams")
    ap.add_argument("--latency", action="store_true", help="paper-comparable single-polynomial latency mode")
    ap.add_argument("--automorph", action="store_true", help="SURVEY f4 automorph bandwidth mode")
    ap.add_argument("--extprod", action="store_true", help="SURVEY f1 TFHE external product mode")
    ap.add_argument("--modup", action="store_true", help="SURVEY f2 CKKS ModUp (INTT -> BConv -> NTT) mode")
    ap.add_argument("--keyswitch", action="store_true", help="SURVEY f2 CKKS key switch / HROT mode")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
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
    elif args.impl == "reference":
        bench_reference(args, wl, parts)
    else:
        bench_ours(args, wl, parts)


if __name__ == "__main__":
    main()
