import os, sys
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import p2p_inputs as G
import paper_2511_21535_b200 as P
inp = G.plummer_tiles(12_500_000, 256, 1, 0)
pos = torch.from_numpy(inp.pos).cuda(); m = torch.from_numpy(inp.mass).cuda()
phi = torch.empty(inp.n, device="cuda"); field = torch.empty((inp.n, 3), device="cuda")
comm = P.p2p_comm_create(1, 0, P.p2p_comm_unique_id())
for _ in range(2):
    with P.Plan(P.P2P_GRAVITY, pos, m, inp.h, inp.lo, inp.nbox, inp.periodic, eps=inp.eps, comm=comm) as pl:
        pl.restructure(); pl.eval(P.P2P_REDUNDANT, phi, field)
    torch.cuda.synchronize()
P.p2p_comm_destroy(comm)
