"""Pinned host <-> device copy bandwidth on this box: H2D alone, D2H alone, both
directions at once (two streams), for the cfg5 per-step volume (157.8 MB each way)."""
import json
import torch

n = 157_810_688 // 8
h_in = torch.empty(n, dtype=torch.int64).pin_memory()
h_out = torch.empty(n, dtype=torch.int64).pin_memory()
d_in = torch.empty(n, dtype=torch.int64, device="cuda")
d_out = torch.empty(n, dtype=torch.int64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
res = {}


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d():
    d_in.copy_(h_in, non_blocking=True)


def d2h():
    h_out.copy_(d_out, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = timed(fn)
    res[name] = {"ms": ms, "GBps_per_direction": n * 8 / ms / 1e6}
print(json.dumps(res))
