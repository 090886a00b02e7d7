"""Per-kernel device times of warm bench steps (CUPTI via torch.profiler: no serialisation, no clock lock).
One step = p2p_plan_update + p2p_restructure + p2p_eval(REDUNDANT) on a persistent plan, like bench.py.
usage: python scripts/kprof.py [workload] [steps] [layouts, e.g. redundant,indexed]"""
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import p2p_inputs as G  # noqa: E402
import paper_2511_21535_b200 as P  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c5w"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 5
LAYS = sys.argv[3].split(",") if len(sys.argv) > 3 else ["redundant"]
base, _, t_ad = wl.partition("-adaptive-t")  # e.g. c3-adaptive-t4: adaptive leaves of threshold t (bench.py)
inp = G.plummer_tiles(12_500_000, 256, 1, 0) if base == "c5w" else G.config(base)
pos = torch.from_numpy(inp.pos).cuda()
m = torch.from_numpy(inp.mass).cuda()
phi = torch.empty(inp.n, device="cuda")
field = torch.empty((inp.n, 3), device="cuda")
# P2P_KPROF_COMM=1: the collective (multi-GPU) plan path with a 1-rank NCCL communicator
comm = P.p2p_comm_create(1, 0, P.p2p_comm_unique_id()) if os.environ.get("P2P_KPROF_COMM") else None
plan = P.Plan(P.P2P_GRAVITY, pos, m, inp.h, inp.lo, inp.nbox, inp.periodic, eps=inp.eps, comm=comm)
if t_ad:
    plan.enable_adaptive(int(t_ad))


def step():
    plan.update(pos, m)
    plan.restructure()
    for lay in LAYS:
        plan.eval(P.LAYOUTS[lay], phi, field)


for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(K):
        step()
    torch.cuda.synchronize()
acc = collections.defaultdict(list)
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        name = e.name.replace("(anonymous namespace)::", "").split("(")[0].replace("void ", "").replace("p2p::", "")
        acc[name[:80]].append(e.device_time)
tot = 0.0
for name, v in acc.items():
    per = sum(v) / K
    tot += per
    print(f"{per:9.1f} us/step  x{len(v) // K:<3d} {name}")
print(f"{tot:9.1f} us/step  total ({wl}, {K} steps)")
plan.close()
if comm is not None:
    P.p2p_comm_destroy(comm)
