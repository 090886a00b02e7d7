"""SURVEY NEXT-1 measurement: the adaptive-leaf path (p2p_adaptive_eval: leaves, closed lists, redundant runs,
REDUNDANT eval, and the INDEXED baseline on the same leaves) on BASELINE configs[2]'s clustered 10^6 Plummer input (128^3 finest boxes, periodic) for several
clustering thresholds t, next to the uniform-grid path on the same plan.  Kernel times from CUPTI (torch.profiler,
warm, no serialisation); pairs from the returned CSR.  Prints one JSON line per t.
usage: python scripts/bench_adaptive.py [t,t,...]"""
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import p2p_inputs as G  # noqa: E402
import paper_2511_21535_b200 as P  # noqa: E402

ts = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "8,16,64").split(",")]
inp = G.config("c3")
pos = torch.from_numpy(inp.pos).cuda()
m = torch.from_numpy(inp.mass).cuda()
phi = torch.empty(inp.n, device="cuda")
fld = torch.empty((inp.n, 3), device="cuda")
peak = 148 * 128 * 1965e6 / 13


def kernel_times(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
    acc = collections.defaultdict(float)
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            name = e.name.replace("(anonymous namespace)::", "").split("(")[0].replace("void ", "").replace("p2p::", "")
            acc[name.split("<")[0]] += e.device_time / reps
    return acc


with P.Plan(P.P2P_GRAVITY, pos, m, inp.h, inp.lo, inp.nbox, inp.periodic, eps=inp.eps) as plan:
    info = plan.info
    plan.restructure()
    grid = kernel_times(lambda: (plan.restructure(), plan.eval(P.P2P_REDUNDANT, phi, fld)))
    I_grid = int(info.n_pairs)
    for t in ts:
        ln, px, st = P.p2p_adaptive_leaves(plan.handle, t, 9, info.n_boxes)
        off, nbr, code = P.p2p_adaptive_neighbours(plan.handle, t, 9, info.n_boxes + 1, 27 * 64 * info.n_boxes)
        cnt = np.diff(np.append(st.astype(np.int64), inp.n))
        I = int(sum(cnt[a] * cnt[nbr[off[a]:off[a + 1]]].sum() for a in range(len(cnt))))
        k = kernel_times(lambda: P.p2p_adaptive_eval(plan.handle, t, 9, phi.data_ptr(), fld.data_ptr()))
        ki = kernel_times(lambda: P.p2p_adaptive_eval(plan.handle, t, 9, phi.data_ptr(), fld.data_ptr(),
                                                      layout=P.P2P_INDEXED))
        ev_idx = ki.get("k_eval_gravity", 0.0) * 1e-6
        ev = k.get("k_eval_gravity", 0.0) * 1e-6
        rs = k.get("k_adapt_restructure_chunks", 0.0) * 1e-6
        build = sum(v for n, v in k.items() if n in ("k_leaf_len", "k_dil_ranges", "k_dil_fill", "k_dil_merge", "k_leaf_keys", "k_scan_reduce",
                                                       "k_scan_partials", "k_scan_down", "k_adapt_count",
                                                       "k_adapt_items")) * 1e-6
        print(json.dumps({"workload": "c3 (10^6 Plummer, 128^3 finest boxes)", "t": t, "leaves": len(cnt),
                          "max_leaf": int(cnt.max()), "entries": int(len(nbr)), "pairs": I,
                          "eval_ms": ev * 1e3, "restructure_ms": rs * 1e3, "structure_kernels_ms": build * 1e3,
                          "eval_pairs_per_s": I / ev if ev else None, "eval_frac_fp32": I / ev / peak if ev else None,
                          "restr_plus_eval_pairs_per_s": I / (ev + rs) if ev else None,
                          "indexed_eval_ms": ev_idx * 1e3, "redundant_kernel_vs_indexed": ev_idx / ev if ev else None,
                          "redundant_e2e_vs_indexed": ev_idx / (ev + rs) if ev else None,
                          "grid_pairs": I_grid, "grid_eval_ms": grid.get("k_eval_gravity", 0) * 1e-3,
                          "grid_restructure_ms": grid.get("k_restructure_gravity", 0) * 1e-3,
                          "kernels_us": {n: round(v, 1) for n, v in k.items()}}), flush=True)
