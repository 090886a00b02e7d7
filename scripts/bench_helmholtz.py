"""Helmholtz (DBIM-like, BASELINE configs[1]) timing: plan (one-off geometry), restructure (im2col Xg), eval
REDUNDANT / INDEXED, as pair-interactions (complex MACs) per second.  Rooflines: the CUDA-core kernels against the
FP32 pipe (4 FFMA per complex MAC: peak = n_SM * 128 * f_max / 4); the fp32 REDUNDANT eval (t in {16, 64}) is the
3xTF32 tensor-core GEMM (k_helm_tc.cu) -- 3 TF32 MMAs x 8 real flops per complex MAC against the TF32 dense peak
(MEASURED_PEAKS bf16 x the nominal TF32 / BF16 ratio 1.1 / 2.25).  Prints one JSON line per workload.
usage: python scripts/bench_helmholtz.py [c2a|c2b ...]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import p2p_inputs as G  # noqa: E402
import paper_2511_21535_b200 as P  # noqa: E402
from bench import ClockSampler  # noqa: E402  (nvidia-smi clocks + throttle reasons during the timed region)


def timed(fn, stream, reps=10):
    flush = torch.empty(128 * 2**20, dtype=torch.float32, device="cuda")
    ts = []
    for _ in range(reps + 3):
        flush.add_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts[3:]))


def main():
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"sm_max_mhz": 1965.0, "hbm_gbs": 6650.0}
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    for wl in (sys.argv[1:] or ["c2a", "c2b"]):
        inp = G.config(wl)
        stream = torch.cuda.current_stream()
        xr = torch.from_numpy(inp.x.view(np.float32).reshape(-1, 2)).cuda()
        pos = torch.from_numpy(inp.pos).cuda()
        y = torch.empty((inp.n, 2), dtype=torch.float32, device="cuda")
        with P.Plan(P.P2P_HELMHOLTZ2D, pos, xr, inp.h, inp.lo, inp.nbox, 0, k=inp.k, t=inp.t) as plan:
            with ClockSampler(0) as clk:
                # enough repetitions that the 50 ms clock sampler sees the timed region
                t_rest = timed(plan.restructure, stream, reps=200)
                t_red = timed(lambda: plan.eval(P.P2P_REDUNDANT, y), stream, reps=200)
                t_idx = timed(lambda: plan.eval(P.P2P_INDEXED, y), stream, reps=200)
            info = plan.info
        I = int(info.n_pairs)
        peak = nsm * 128 * peaks["sm_max_mhz"] * 1e6 / 4
        tf32_peak = peaks.get("bf16_tflops", 2250.0) * 1e12 * (1.1 / 2.25)
        tc = inp.t in (16, 64) and os.environ.get("P2P_HELM_SIMT", "0") != "1"
        xg_bytes = int(info.n_red) * 8
        out = {"workload": wl, "N": inp.n, "t": inp.t, "boxes": int(info.n_boxes), "pairs": I,
               "restructure_ms": t_rest, "eval_redundant_ms": t_red, "eval_indexed_ms": t_idx,
               "eval_pairs_per_s": I / (t_red * 1e-3), "eval_frac_fp32": I / (t_red * 1e-3) / peak,
               "eval_path": "tcgen05 3xTF32 GEMM" if tc else "CUDA-core FP32x2",
               "eval_tensor_tflops": (24.0 * I / (t_red * 1e-3) / 1e12) if tc else None,
               "eval_frac_tf32_peak": (24.0 * I / (t_red * 1e-3) / tf32_peak) if tc else None,
               "indexed_frac_fp32": I / (t_idx * 1e-3) / peak,
               "restructure_plus_eval_pairs_per_s": I / ((t_rest + t_red) * 1e-3),
               "indexed_pairs_per_s": I / (t_idx * 1e-3),
               "restructure_hbm_frac": (xg_bytes + inp.n * 8) / (t_rest * 1e-3) / (peaks["hbm_gbs"] * 1e9),
               "peak_basis": f"{nsm} SM x 128 FP32 lanes x {peaks['sm_max_mhz']} MHz / 4 FFMA per complex MAC",
               "clocks": clk.summary()}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
