"""e2e variants for cfg5: parts concurrent on two streams vs sequential on one."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import inputs
import paper_2410_05934_b200 as R
from bench import WORKLOADS, primes_for

parts = WORKLOADS["cfg5"]["parts"]
states = []
for (logn, limbs, polys, seed) in parts:
    mods = primes_for(logn, limbs)
    plan = R.Plan(logn, mods)
    a = inputs.residues(seed, polys, mods, 1 << logn)
    ha = torch.from_numpy(a.view(np.int64)).pin_memory()
    hc = torch.empty_like(ha).pin_memory()
    ws = torch.empty(ha.shape, dtype=torch.int64, device="cuda")
    b = torch.from_numpy(inputs.residues(seed + 1, polys, mods, 1 << logn).view(np.int64)).cuda()
    states.append(dict(plan=plan, ha=ha, hc=hc, ws=ws, b=b))
main = torch.cuda.current_stream()
ss = [torch.cuda.Stream() for _ in states]


def conc():
    ev = torch.cuda.Event(); ev.record(main)
    for s, st in zip(states, ss):
        st.wait_event(ev)
        R.execute_host(s["plan"], R.OP_POLYMUL_EVAL, s["hc"], s["ha"], s["ws"], b_dev=s["b"], stream=st)
    for st in ss:
        main.wait_stream(st)


def seq(order=(1, 0)):
    for i in order:
        s = states[i]
        R.execute_host(s["plan"], R.OP_POLYMUL_EVAL, s["hc"], s["ha"], s["ws"], b_dev=s["b"], stream=main)


def big_only():
    s = states[1]
    R.execute_host(s["plan"], R.OP_POLYMUL_EVAL, s["hc"], s["ha"], s["ws"], b_dev=s["b"], stream=main)


for name, f in (("concurrent", conc), ("seq_10", seq), ("seq_01", lambda: seq((0, 1))), ("big_only", big_only)):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"{name:12s} {ms:.3f} ms/step  e2e {32858 / (ms * 1e-3):.3e}")
