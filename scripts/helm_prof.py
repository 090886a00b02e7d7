"""ncu target: the Helmholtz tensor-core GEMM on configs[1] (c2a / c2b), REDUNDANT (Xg by TMA) then INDEXED
(tensor-core gather).  usage: python scripts/helm_prof.py [c2a|c2b]"""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import p2p_inputs as G  # noqa: E402
import paper_2511_21535_b200 as P  # noqa: E402

inp = G.config(sys.argv[1] if len(sys.argv) > 1 else "c2b")
xr = torch.from_numpy(inp.x.view(np.float32).reshape(-1, 2)).cuda()
with P.Plan(P.P2P_HELMHOLTZ2D, torch.from_numpy(inp.pos).cuda(), xr, inp.h, inp.lo, inp.nbox, 0, k=inp.k,
            t=inp.t) as plan:
    plan.restructure()
    plan.eval(P.P2P_REDUNDANT)
    plan.eval(P.P2P_INDEXED)
    torch.cuda.synchronize()
