"""bench.py -- P2P pair-interactions/s of the B200-native near-field operator (BASELINE.json metric).

One "step" = one pass of the whole hot path over one batch of synthetic input, exactly what a PhotoNs-like time
step does (the tree is rebuilt every step): p2p_plan_create (a1 bin + Morton key, a2 radix sort, a3
permute, a4 box scan, a5 neighbour CSR) -> p2p_restructure (a6 redundant gather) -> p2p_eval(P2P_REDUNDANT)
(a7 gravity P2P + a9 scatter) -> p2p_destroy.  value = pair interactions I of the whole job / device time.

Workload (default `c5w`): BASELINE configs[4]'s per-GPU weak-scaling tile -- a Plummer cluster (a = 0.1 tile) of
12.5M particles in 256^3 periodic leaf boxes per GPU; N GPUs = N tiles (1x1x1, 2x1x1, 2x2x1, 2x2x2), each rank
owning one tile.  Inputs (200 MB) and the redundant buffer (4.75 GB) exceed the 126 MB L2, and L2
is additionally flushed between timed steps.

Extra keys beside the driver contract: "phases" (plan / restructure / eval split, kernel-only and
restructure+eval rates, the INDEXED comparison), "roofline_hbm" (restructure vs HBM).
`--impl reference` times the fp64 CPU oracle (oracle/, as it stands) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BASELINE = json.load(open(os.path.join(ROOT, "BASELINE.json")))
METRIC = BASELINE["metric"]
UNIT = "pair-interactions/s"
FP32_INSTR_PER_PAIR = 13           # SURVEY §8d, verified from SASS
FP64_INSTR_PER_PAIR = 18           # fp64 hot loop SASS per pair: 3 DADD + 3 DFMA (r^2) + 5 (rsqrt, C14: MUFU.RSQ64H
                                   # seed + DMUL/DFMA second-order Newton step) + 3 DMUL + 1 DADD + 3 DFMA (
                                   # 26 with the correctly rounded 1/sqrt of round 2's first fp64 line)
FP64_LANES_PER_SM = 64             # DFMA lane-ops per clock per SM, measured (profiles/r02_ubench_fp64.txt)
SM_COUNT_NOMINAL = 148
LANES_PER_SM = 128


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "sm_max_mhz": d.get("sm_max_mhz", 1965.0), "src": "measured"}
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "src": "fallback"}


# ------------------------------------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 50 ms during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active"
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi takes a few hundred ms to start: wait for its first sample so that the timed region
            # (which may last only ~0.2 s) is covered
            t0 = time.time()
            while not self.samples and time.time() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.01)
            self.n_before = len(self.samples)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 4:
                try:
                    self.samples.append((float(parts[0]), float(parts[1]), parts[2], int(parts[3], 16)))
                except ValueError:
                    pass

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        timed = self.samples[max(0, getattr(self, "n_before", 1) - 1):]  # the last pre-region sample onwards
        load = [s for s in timed if not (s[3] & 0x1)] or timed
        reasons = set()
        for s in load:
            for bit, name in self.REASONS.items():
                if s[3] & bit:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(s[0] for s in load), "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": sorted(reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------------------------------------ workload
def make_workload(name: str, rank: int, world: int, seed: int = 0, dtype=np.float32):
    import p2p_inputs as G
    if "-adaptive-t" in name:  # e.g. c3-adaptive-t16: the base workload on adaptive leaves of threshold t (NEXT-1)
        base, t = name.split("-adaptive-t")
        inp, desc = make_workload(base, rank, world, seed, dtype)
        return inp, f"{desc} on adaptive binary-tree leaves, clustering threshold t = {int(t)} (p2p_adaptive_enable)"
    if name == "c5w":
        # rank r owns tile r of the G-tile domain (Morton octant == tile for 2x2x2)
        inp = G.plummer_tiles(12_500_000, 256, world, seed, dtype=dtype, tile_index=rank)
        return inp, f"c5w: Plummer tile (a=0.1 tile) 12.5M particles/GPU, 256^3 boxes/tile, {world} tile(s)"
    return G.config(name, seed, dtype), name


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c5w")
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"],
                    help="fp64: the same workload in double precision end to end (P:L258's 8-byte fields)")
    ap.add_argument("--comm", default="nccl", choices=["nccl", "ipc"],
                    help="N > 1: the NCCL communicator (one process per GPU) or the CUDA-IPC peer-memory one "
                         "(p2p_comm_create_ipc; also runs N processes on ONE GPU -- not a scaling measurement)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return reference_arm(args, rank, world)
    return ours(args, rank, world, local)


# ------------------------------------------------------------------------------------------------ our arm
def ours(args, rank, world, local):
    import torch
    import paper_2511_21535_b200 as P

    assert torch.cuda.is_available(), "bench.py needs a CUDA device"
    ipc = args.comm == "ipc" and world > 1
    ndev = torch.cuda.device_count()
    if ipc:
        local = local % ndev   # IPC ranks may share a device (more processes than GPUs)
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if ipc:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    red_dev = torch.device("cpu") if ipc else dev   # where the timing reductions run (gloo: host tensors)
    W = max(3, args.warmup)
    K = max(1, args.steps)

    f64 = args.precision == "fp64"
    fdt = torch.float64 if f64 else torch.float32
    inp, wdesc = make_workload(args.workload, rank, world, dtype=np.float64 if f64 else np.float32)
    pos_h = torch.from_numpy(inp.pos).pin_memory()
    m_h = torch.from_numpy(inp.mass).pin_memory()
    pos = pos_h.to(dev)
    m = m_h.to(dev)
    N = inp.n
    stream = torch.cuda.current_stream()
    flush = torch.empty(int(512 * 2**20) // 4, dtype=torch.float32, device=dev)   # 512 MB > 126 MB L2

    def l2_flush():
        flush.add_(1.0)

    phi = torch.empty(N, dtype=fdt, device=dev)
    field = torch.empty((N, 3), dtype=fdt, device=dev)

    comm = None
    if world > 1 and ipc:
        # CUDA-IPC communicator: rank 0 draws the rendezvous token, broadcast over the gloo group
        import secrets
        tok = [("p2pbench_" + secrets.token_hex(8)) if rank == 0 else None]
        dist.broadcast_object_list(tok, 0)
        comm = P.p2p_comm_create_ipc(world, rank, tok[0])
    elif world > 1:
        # NCCL communicator owned by libp2p; rank 0's unique id is broadcast over the torch process group
        idt = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(P.p2p_comm_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        comm = P.p2p_comm_create(world, rank, bytes(idt.cpu().numpy().tobytes()))

    # one persistent plan = the simulation's setup (allocations); every step rebuilds a1..a5 from the positions
    # with p2p_plan_update (1 GPU: asynchronous, no host sync, no allocation), then a6, a7+a9.
    # N GPUs: the update is collective (histogram all-reduce + repartition + halo exchange over NCCL, whose
    # sizes need host syncs, then a1..a5 on the plan's buffers), a6, a7+a9 and the reverse all-to-all-v.
    splan = P.Plan(P.P2P_GRAVITY, pos, m, inp.h, inp.lo, inp.nbox, inp.periodic, eps=inp.eps, stream=stream,
                   comm=comm)
    if "-adaptive-t" in args.workload:
        # adaptive-leaf mode: the same step over the leaves, asynchronous (measured once here)
        splan.enable_adaptive(int(args.workload.split("-adaptive-t")[1]))
    holder = {"plan": splan}

    def step(events=None):
        ev = events
        if ev:
            ev[0].record(stream)
        splan.update(pos, m)   # N > 1: collective (repartition + halo exchange over NCCL, then a1..a5)
        plan = holder["plan"]
        if ev:
            ev[1].record(stream)
        plan.restructure()
        if ev:
            ev[2].record(stream)
        plan.eval(P.P2P_REDUNDANT, phi, field)
        if ev:
            ev[3].record(stream)

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(W):
        step()
        l2_flush()
    barrier()
    I = int(holder["plan"].refresh_info().n_pairs)

    # ---- timed region: K full steps, L2 flushed between steps (outside the events) ----
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K)]
    launches0 = P.p2p_kernel_launch_count()
    with ClockSampler(local) as clk:
        barrier()
        for k in range(K):
            step(evs[k])
            l2_flush()
        barrier()
    launches = P.p2p_kernel_launch_count() - launches0
    t_plan = [e[0].elapsed_time(e[1]) for e in evs]
    t_rest = [e[1].elapsed_time(e[2]) for e in evs]
    t_eval = [e[2].elapsed_time(e[3]) for e in evs]
    t_step = [e[0].elapsed_time(e[3]) for e in evs]
    ms_step = float(np.mean(t_step))
    if dist:
        t = torch.tensor([ms_step], device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
        tot = torch.tensor([float(I)], device=red_dev, dtype=torch.float64)
        dist.all_reduce(tot)
        I_all = int(tot.item())
    else:
        I_all = I
    value = I_all / (ms_step * 1e-3)

    # ---- kernel-only phases on a persistent plan (same stream, L2 flushed before each launch) ----
    plan = holder["plan"]
    plan.restructure()

    def timed(fn, reps):
        ts = []
        for _ in range(reps):
            l2_flush()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        return float(np.median(ts)), float(np.min(ts))

    reps = max(3, K)
    t_ev_red = timed(lambda: plan.eval(P.P2P_REDUNDANT, phi, field), reps)
    t_ev_idx = timed(lambda: plan.eval(P.P2P_INDEXED, phi, field), reps)
    t_restr = timed(lambda: plan.restructure(), reps)
    R = int(plan.info.n_red)
    B = int(plan.info.n_boxes)

    pk = peaks()
    # roofline of the dominant kernel (eval): FP32-pipe bound, 13 FP32 instructions per pair;
    # fp64: FP64-pipe bound, FP64_INSTR_PER_PAIR FP64-pipe instructions per pair (SASS hot loop) at the measured DFMA rate per SM
    # (scripts/ubench_fp64.cu, profiles/r02_ubench_fp64.txt)
    eval_ms_in_step = float(np.mean(t_eval))
    achieved = I / (eval_ms_in_step * 1e-3)
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    lanes = FP64_LANES_PER_SM if f64 else LANES_PER_SM
    ipp = FP64_INSTR_PER_PAIR if f64 else FP32_INSTR_PER_PAIR
    peak_pairs = n_sm * lanes * pk["sm_max_mhz"] * 1e6 / ipp
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_eval_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get(args.workload)
        except (ValueError, OSError):
            traffic = None
    # restructure vs HBM: writes 16 R bytes + compulsory reads 16 N_src (= 16 N) bytes
    rb = 32 if f64 else 16   # record bytes (float4 / double4)
    rest_bytes = rb * R + rb * N
    rest_ms = float(np.mean(t_rest))
    # SURVEY §8d end-to-end roofline: the FP32-bound eval time + the HBM-bound restructure time over the measured
    # restructure + eval time of the step
    t_roof = (I / peak_pairs + rest_bytes / (pk["hbm_gbs"] * 1e9)) * 1e3

    out = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": K,
        "warmup": W,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64" if f64 else "f32",
        "data": "synthetic (seeded numpy PCG64 Plummer tiles; BASELINE configs[4] per-GPU tile)",
        "config": {"workload": wdesc, "N_per_gpu": N, "boxes_per_gpu": B, "pairs_per_gpu_per_step": I,
                   "red_records_per_gpu": R, "parallelism": (f"morton-range sharding over {world} GPUs: NCCL histogram all-reduce + all-to-all-v "
                                   f"repartition + halo exchange (one Plummer tile per GPU)") if world > 1 and not ipc
                   else (f"morton-range sharding over {world} processes on {min(world, ndev)} GPU(s) through the "
                         f"CUDA-IPC peer-memory communicator" + (" -- several ranks share a GPU: NOT a scaling "
                                                                   "measurement" if world > ndev else ""))
                   if ipc else "1 GPU",
                   "l2": "inputs+red buffer > L2 and 512 MB L2 flush between timed steps",
                   "step": "p2p_plan_update(a1-a5) + p2p_restructure(a6) + p2p_eval REDUNDANT(a7,a9); plan created once"},
        "roofline": {"bound": "alu", "kernel": f"k_eval_gravity<{'double' if f64 else 'float'},REDUNDANT,"
                                                     f"{2 if f64 else 4}>", "achieved": achieved / 1e9,
                     "peak": peak_pairs / 1e9,
                     "unit": f"Gpair/s ({'FP64' if f64 else 'FP32'} pipe: {ipp} instr/pair)",
                     "frac": achieved / peak_pairs, "traffic": traffic if not f64 else None,
                     "peak_basis": f"{n_sm} SMs x {lanes} {'FP64 (measured DFMA rate)' if f64 else 'FP32'} lanes x "
                                   f"{pk['sm_max_mhz']:.0f} MHz ({pk['src']}) / {ipp}"},
        "roofline_e2e": {"frac": t_roof / (rest_ms + eval_ms_in_step), "t_roofline_ms": t_roof,
                         "t_measured_ms": rest_ms + eval_ms_in_step,
                         "formula": "SURVEY 8d: (ipp I / (n_SM lanes f) + (rb R + rb N) / BW_hbm) / (t_restructure + "
                                    "t_eval), ipp = pipe instructions per pair, rb = record bytes"},
        "roofline_hbm": {"kernel": f"k_restructure_gravity<{'double' if f64 else 'float'}>", "bound": "hbm",
                         "unit": "GB/s",
                         "achieved": rest_bytes / (rest_ms * 1e-3) / 1e9, "peak": pk["hbm_gbs"],
                         "frac": rest_bytes / (rest_ms * 1e-3) / 1e9 / pk["hbm_gbs"], "bytes": rest_bytes},
        "phases": {
            "update_a1_a5_ms": float(np.mean(t_plan)), "restructure_ms": rest_ms, "eval_ms": eval_ms_in_step,
            "kernel_only_pairs_per_s": I / (t_ev_red[0] * 1e-3),
            "restructure_plus_eval_pairs_per_s": I / ((t_restr[0] + t_ev_red[0]) * 1e-3),
            "indexed_eval_pairs_per_s": I / (t_ev_idx[0] * 1e-3),
            "eval_redundant_ms_median_min": t_ev_red, "eval_indexed_ms_median_min": t_ev_idx,
            "restructure_ms_median_min": t_restr,
            "redundant_e2e_vs_indexed": t_ev_idx[0] / (t_restr[0] + t_ev_red[0]),
            "redundant_kernel_vs_indexed": t_ev_idx[0] / t_ev_red[0],
        },
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }

    # ---- e2e: the public API with HOST buffers (H2D of inputs + D2H of results inside the timed region) ----
    if not args.no_e2e:
        if comm is None:
            # the time-stepping user's call sequence on the persistent plan, through the host-buffer ABI:
            # H2D of the step's inputs (pinned) + a1..a5, a6, a7+a9 + D2H of phi and field, every step
            phi_h = torch.empty(N, dtype=fdt, pin_memory=True)
            field_h = torch.empty((N, 3), dtype=fdt, pin_memory=True)
            api = "Plan.update_host + restructure + eval_host (p2p_plan_update_host / p2p_eval_host, pinned)"

            def e2e_call():
                splan.update_host(pos_h, m_h)
                splan.restructure()
                splan.eval_host(P.P2P_REDUNDANT, phi_h, field_h)
        else:
            # collective plans have no host-buffer entry points: the same sequence with the copies done by torch
            # on the plan's stream (pinned buffers, non_blocking)
            phi_h = torch.empty(N, dtype=fdt, pin_memory=True)
            field_h = torch.empty((N, 3), dtype=fdt, pin_memory=True)
            pos_e = torch.empty_like(pos)
            m_e = torch.empty_like(m)
            api = "H2D (pinned) + collective Plan.update + restructure + eval + D2H (persistent plan)"

            def e2e_call():
                pos_e.copy_(pos_h, non_blocking=True)
                m_e.copy_(m_h, non_blocking=True)
                splan.update(pos_e, m_e)
                splan.restructure()
                splan.eval(P.P2P_REDUNDANT, phi, field)
                phi_h.copy_(phi, non_blocking=True)
                field_h.copy_(field, non_blocking=True)

        def e2e_once():
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            e2e_call()
            b.record(stream)
            b.synchronize()
            return a.elapsed_time(b)
        e2e_once()
        te = float(np.median([e2e_once() for _ in range(max(2, min(K, 5)))]))
        if dist:
            t = torch.tensor([te], device=red_dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te = float(t.item())
        out["e2e"] = {"value": I_all / (te * 1e-3), "unit": UNIT, "ms_per_step": te,
                      "h2d_bytes_per_step": int((pos_h.numel() + m_h.numel()) * pos_h.element_size()),
                      "d2h_bytes_per_step": int(N * 4 * phi_h.element_size()), "api": api}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(inp, budget_s=12.0)
    holder["plan"].close()
    if comm is not None:
        P.p2p_comm_destroy(comm)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(out), flush=True)


# ------------------------------------------------------------------------------------------------ oracle
def _oracle_sample(gp, target_pairs: float, seed: int = 1):
    """a seeded random sample of target boxes whose pair count is about target_pairs (evaluated by the fp64
    oracle's plain-definition mode ii)."""
    rng = np.random.default_rng(seed)
    order = rng.permutation(gp.B)
    nb = np.diff(gp.bstart.astype(np.int64))
    nsrc = np.diff(gp.red_off.astype(np.int64))
    cum = np.cumsum(nb[order] * nsrc[order])
    k = int(np.searchsorted(cum, target_pairs)) + 1
    sel = np.sort(order[:min(k, gp.B)])
    return sel, int((nb[sel] * nsrc[sel]).sum())


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(inp, budget_s: float = 12.0):
    """the fp64 oracle (mode ii) on seeded-random target-box samples of the workload: all host cores (the
    reported value) and 1 core (SURVEY §8d asks for both)"""
    import oracle
    gp = oracle.GravityPlan(inp, with_red=False)
    ncpu = os.cpu_count()

    def run(threads, budget):
        used = oracle.set_threads(threads)
        sel, pairs = _oracle_sample(gp, 5e7 / max(1, ncpu // threads))
        t0 = time.perf_counter()
        gp.eval_indexed_boxes(sel)
        rate = pairs / (time.perf_counter() - t0)
        # scale the sample to about `budget` s of wall time, then time it
        sel, pairs = _oracle_sample(gp, min(rate * budget, float(gp.I)), seed=2)
        t0 = time.perf_counter()
        gp.eval_indexed_boxes(sel)
        dt = time.perf_counter() - t0
        return used, sel, pairs, dt

    used1, sel1, pairs1, dt1 = run(1, budget_s / 2)
    used, sel, pairs, dt = run(ncpu, budget_s)
    oracle.set_threads(ncpu)
    what = "all" if len(sel) >= gp.B else "seeded-random"
    return {"value": pairs / dt, "unit": UNIT, "cores": used, "kind": "oracle",
            "cpu": cpu_model(),
            "one_core": {"value": pairs1 / dt1, "cores": used1,
                         "sample": f"{len(sel1)} seeded-random target boxes ({pairs1} pairs, {dt1:.1f} s)"},
            "sample": f"fp64 oracle mode (ii) over {what} {len(sel)} target boxes ({pairs} pairs, {dt:.1f} s wall, "
                      f"OpenMP {used} threads = {dt * used:.0f} core-s) of the same workload; "
                      f"structure build excluded; one_core = the same oracle on 1 thread"}


def reference_arm(args, rank, world):
    if rank != 0:
        return
    inp, wdesc = make_workload(args.workload, 0, world)
    import oracle
    gp = oracle.GravityPlan(inp, with_red=False)
    # per step: ~5e8 pairs (a few seconds on the host cores), so --steps K --warmup W ends within minutes
    sel, pairs = _oracle_sample(gp, 5e8, seed=3)
    for _ in range(args.warmup):
        gp.eval_indexed_boxes(sel)
    ts = []
    for _ in range(max(1, args.steps)):
        t0 = time.perf_counter()
        gp.eval_indexed_boxes(sel)
        ts.append(time.perf_counter() - t0)
    ms = 1e3 * float(np.mean(ts))
    v = pairs / (ms * 1e-3)
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": wdesc, "sample_pairs_per_step": pairs, "sample_boxes": int(len(sel))},
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle", "cpu": cpu_model(),
                            "sample": f"{len(sel)} seeded-random target boxes ({pairs} pairs) per step, fp64 mode ii"},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
