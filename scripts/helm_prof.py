import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import p2p_inputs as G
import paper_2511_21535_b200 as P
inp = G.config("c2b")
xr = torch.from_numpy(inp.x.view(np.float32).reshape(-1, 2)).cuda()
with P.Plan(P.P2P_HELMHOLTZ2D, torch.from_numpy(inp.pos).cuda(), xr, inp.h, inp.lo, inp.nbox, 0, k=inp.k, t=inp.t) as plan:
    plan.restructure()
    for _ in range(2):
        y = plan.eval(P.P2P_REDUNDANT)
    torch.cuda.synchronize()
