"""host-side timing of plan creation (P2P_TRACE=1 prints the library's own phase stamps)"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import p2p_inputs as G
import paper_2511_21535_b200 as P
wl = sys.argv[1] if len(sys.argv) > 1 else "c5w"
inp = G.plummer_tiles(12_500_000, 256, 1, 0) if wl == "c5w" else G.config(wl)
pos = torch.from_numpy(inp.pos).cuda(); m = torch.from_numpy(inp.mass).cuda()
for it in range(4):
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); a.record()
    plan = P.Plan(P.P2P_GRAVITY, pos, m, inp.h, inp.lo, inp.nbox, inp.periodic, eps=inp.eps)
    b.record(); t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"iter {it}: host {1e3*(t1-t0):.2f} ms, device-events {a.elapsed_time(b):.2f} ms", file=sys.stderr)
    plan.restructure(); plan.eval(P.P2P_REDUNDANT)
    t2 = time.perf_counter(); plan.close(); torch.cuda.synchronize(); print(f"  close {1e3*(time.perf_counter()-t2):.2f} ms", file=sys.stderr)
