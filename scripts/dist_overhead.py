"""Per-step cost of the collective (multi-GPU) plan path at G = 1 (NCCL, one rank) vs the single-GPU
persistent-plan update, on one workload: what the N > 1 bench pays for re-creating the plan every step.
usage: python scripts/dist_overhead.py [workload]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import p2p_inputs as G  # noqa: E402
import paper_2511_21535_b200 as P  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c5w"
inp = G.plummer_tiles(12_500_000, 256, 1, 0) if wl == "c5w" else G.config(wl)
pos = torch.from_numpy(inp.pos).cuda()
m = torch.from_numpy(inp.mass).cuda()
phi = torch.empty(inp.n, device="cuda")
field = torch.empty((inp.n, 3), device="cuda")
st = torch.cuda.current_stream()
comm = P.p2p_comm_create(1, 0, P.p2p_comm_unique_id())


def t_events(fn, reps=5):
    ts = []
    for _ in range(reps + 2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        h0 = time.perf_counter()
        a.record(st)
        fn()
        b.record(st)
        b.synchronize()
        ts.append((a.elapsed_time(b), (time.perf_counter() - h0) * 1e3))
    ts = ts[2:]
    return float(np.median([x[0] for x in ts])), float(np.median([x[1] for x in ts]))


def coll_step():
    with P.Plan(P.P2P_GRAVITY, pos, m, inp.h, inp.lo, inp.nbox, inp.periodic, eps=inp.eps, comm=comm) as pl:
        pl.restructure()
        pl.eval(P.P2P_REDUNDANT, phi, field)


plan = P.Plan(P.P2P_GRAVITY, pos, m, inp.h, inp.lo, inp.nbox, inp.periodic, eps=inp.eps)


def upd_step():
    plan.update(pos, m)
    plan.restructure()
    plan.eval(P.P2P_REDUNDANT, phi, field)


def create_step():
    with P.Plan(P.P2P_GRAVITY, pos, m, inp.h, inp.lo, inp.nbox, inp.periodic, eps=inp.eps) as pl:
        pl.restructure()
        pl.eval(P.P2P_REDUNDANT, phi, field)


cplan = P.Plan(P.P2P_GRAVITY, pos, m, inp.h, inp.lo, inp.nbox, inp.periodic, eps=inp.eps, comm=comm)


def coll_upd_step():
    cplan.update(pos, m)
    cplan.restructure()
    cplan.eval(P.P2P_REDUNDANT, phi, field)


for name, fn in [("update (1-GPU persistent plan)", upd_step), ("create (1-GPU plan per step)", create_step),
                 ("collective update, NCCL 1 rank", coll_upd_step), ("collective create, NCCL 1 rank", coll_step)]:
    dev, wall = t_events(fn)
    print(f"{name:40s} device {dev:8.2f} ms   wall {wall:8.2f} ms", flush=True)
plan.close()
cplan.close()
P.p2p_comm_destroy(comm)
