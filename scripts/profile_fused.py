"""One c5w plan, two p2p_restructure_eval calls (for an ncu capture of the fused kernel)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import p2p_inputs as G  # noqa: E402
import paper_2511_21535_b200 as P  # noqa: E402

inp = G.plummer_tiles(12_500_000, 256, 1, 0)
pos = torch.from_numpy(inp.pos).cuda()
m = torch.from_numpy(inp.mass).cuda()
with P.Plan(P.P2P_GRAVITY, pos, m, inp.h, inp.lo, inp.nbox, inp.periodic, eps=inp.eps) as plan:
    for _ in range(2):
        plan.restructure_eval()
    torch.cuda.synchronize()
print("done")
