"""Run a few bench steps of one workload with nothing else (for ncu launch lists / --set full captures).
usage: python scripts/profile_step.py [workload] [steps] [layouts]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import p2p_inputs as G  # noqa: E402
import paper_2511_21535_b200 as P  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c5w"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
layouts = sys.argv[3].split(",") if len(sys.argv) > 3 else ["redundant"]
base, _, t_ad = wl.partition("-adaptive-t")  # e.g. c3-adaptive-t4: adaptive leaves of threshold t
inp = G.plummer_tiles(12_500_000, 256, 1, 0) if base == "c5w" else G.config(base)
pos = torch.from_numpy(inp.pos).cuda()
m = torch.from_numpy(inp.mass).cuda()
if inp.pos.ndim == 2 and inp.pos.shape[1] == 3:
    for _ in range(steps):
        with P.Plan(P.P2P_GRAVITY, pos, m, inp.h, inp.lo, inp.nbox, inp.periodic, eps=inp.eps) as plan:
            if t_ad:
                plan.enable_adaptive(int(t_ad))
            plan.restructure()
            for lay in layouts:
                plan.eval(P.LAYOUTS[lay])
        torch.cuda.synchronize()
print("done", wl, P.p2p_kernel_launch_count(), "launches")
