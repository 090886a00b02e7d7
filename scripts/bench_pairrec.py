"""SURVEY §8f NEXT-4 measurement: the three redundancy granularities side by side on one B200 --
none (P2P_INDEXED), per target box (P2P_REDUNDANT, the bench's layout) and per interaction pair (P2P_PAIRREC, the
paper's thread-level layout) -- kernel device times from CUPTI (torch.profiler), L2 flushed before every
launch, median over K repetitions; HBM roofline of the pair-record kernels against the measured copy bandwidth.
usage: python scripts/bench_pairrec.py [workloads...]   -> one JSON line per workload"""
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

K = 5
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6546.2, "sm_max_mhz": 1965.0}
HBM = peaks.get("hbm_gbs", 6546.2) * 1e9
FP32_PEAK = 148 * 128 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 13   # pairs/s


def kernel_times(fn, flush):
    """per-kernel device time (us, median over K calls of fn), L2 flushed before each call"""
    acc = collections.defaultdict(list)
    for _ in range(K):
        flush.add_(1.0)
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            fn()
            torch.cuda.synchronize()
        per = collections.defaultdict(float)
        for e in prof.events():
            if e.device_type == torch.autograd.DeviceType.CUDA and "k_" in e.name:
                name = e.name.replace("(anonymous namespace)::", "").split("(")[0].split("<")[0]
                per[name.replace("void ", "").replace("p2p::", "")] += e.device_time
        for k, v in per.items():
            acc[k].append(v)
    return {k: float(np.median(v)) for k, v in acc.items()}


def main():
    wls = sys.argv[1:] or ["c5w", "c4-8", "c4-64", "c3"]
    flush = torch.empty(512 * 2**20 // 4, device="cuda")
    for wl in wls:
        inp = G.plummer_tiles(12_500_000, 256, 1, 0) if wl == "c5w" else G.config(wl)
        pos = torch.from_numpy(inp.pos).cuda()
        m = torch.from_numpy(inp.mass).cuda()
        phi = torch.empty(inp.n, device="cuda")
        field = torch.empty((inp.n, 3), device="cuda")
        with P.Plan(P.P2P_GRAVITY, pos, m, inp.h, inp.lo, inp.nbox, inp.periodic, eps=inp.eps) as plan:
            plan.restructure()
            plan.restructure_pairs()
            nrec, T = P.p2p_get_pairrec_size(plan.handle)
            info = plan.info
            I, R, N = int(info.n_pairs), int(info.n_red), int(info.n_local)
            t = {}
            t.update(kernel_times(plan.restructure, flush))
            t.update(kernel_times(plan.restructure_pairs, flush))
            for lay, tag in ((P.P2P_REDUNDANT, "redundant"), (P.P2P_INDEXED, "indexed")):
                t[f"k_eval_gravity[{tag}]"] = kernel_times(lambda: plan.eval(lay, phi, field), flush)["k_eval_gravity"]
            t.update(kernel_times(lambda: plan.eval(P.P2P_PAIRREC, phi, field), flush))
        out = {"workload": wl, "N": N, "pairs": I, "R": R, "pair_records": nrec, "partial_slots": T,
               "kernel_us": t}
        rs, ev, rd = t.get("k_restructure_pairs", 0), t.get("k_eval_pairrec", 0), t.get("k_reduce_pairrec", 0)
        out["pairrec"] = {
            "restructure_pairs_GBs": 16 * (nrec + N) / (rs * 1e-6) / 1e9 if rs else None,
            "restructure_pairs_hbm_frac": 16 * (nrec + N) / (rs * 1e-6) / HBM if rs else None,
            "eval_pairs_per_s": I / (ev * 1e-6) if ev else None,
            "eval_fp32_frac": I / (ev * 1e-6) / FP32_PEAK if ev else None,
            "reduce_GBs": 16 * (T + N) / (rd * 1e-6) / 1e9 if rd else None,
            "restructure_plus_eval_pairs_per_s": I / ((rs + ev + rd) * 1e-6) if rs else None,
        }
        red = t.get("k_restructure_gravity", 0) + t["k_eval_gravity[redundant]"]
        out["restructure_plus_eval_us"] = {"indexed": t["k_eval_gravity[indexed]"], "redundant": red,
                                           "pairrec": rs + ev + rd}
        print(json.dumps(out), flush=True)
        del pos, m, phi, field
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
