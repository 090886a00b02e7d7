"""Time p2p_restructure_eval against p2p_restructure + p2p_eval(REDUNDANT) and p2p_eval(INDEXED) on one
workload, for several lookahead settings (P2P_OVL_AHEAD, groups of 2^16 records).  CUDA events on the plan
stream, L2 flushed (512 MB write) before every launch, median of 7.  Prints one JSON line per setting.
(needs the p2p_restructure_eval experiment of commit 95157da.)
usage: python scripts/fused_sweep.py [workload] [ahead,ahead,...]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import p2p_inputs as G  # noqa: E402
import paper_2511_21535_b200 as P  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c5w"
aheads = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "2").split(",")]
inp = G.plummer_tiles(12_500_000, 256, 1, 0) if wl == "c5w" else G.config(wl)
pos = torch.from_numpy(inp.pos).cuda()
m = torch.from_numpy(inp.mass).cuda()
flush = torch.empty(128 * 2**20, dtype=torch.float32, device="cuda")
stream = torch.cuda.current_stream()


def timed(fn, reps=7):
    ts = []
    for _ in range(reps):
        flush.add_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


for ahead in aheads:
    os.environ["P2P_OVL_AHEAD"] = str(ahead)
    with P.Plan(P.P2P_GRAVITY, pos, m, inp.h, inp.lo, inp.nbox, inp.periodic, eps=inp.eps) as plan:
        plan.restructure()
        phi, f = plan.eval(P.P2P_REDUNDANT)
        I = plan.info.n_pairs
        t_rs = timed(plan.restructure)
        t_red = timed(lambda: plan.eval(P.P2P_REDUNDANT, phi, f))
        t_idx = timed(lambda: plan.eval(P.P2P_INDEXED, phi, f))
        t_fu = timed(lambda: plan.restructure_eval(phi, f))
        print(json.dumps({"workload": wl, "ahead": ahead, "restructure_ms": t_rs, "eval_red_ms": t_red,
                          "eval_idx_ms": t_idx, "fused_ms": t_fu, "split_ms": t_rs + t_red,
                          "fused_vs_indexed": t_idx / t_fu, "split_vs_indexed": t_idx / (t_rs + t_red),
                          "pairs": I}), flush=True)
