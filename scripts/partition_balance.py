"""Load balance of the multi-GPU Morton-range partition (DESIGN C20), measured with G loopback ranks
on one GPU: for each G, the pair interactions I_r each rank's targets need (= its eval work) and its particle
count (owned + halo).  Prints one JSON line per G: max/mean of I_r (the strong-scaling bound of the eval) and of
the particle counts.  usage: python scripts/partition_balance.py [workload] [G,G,...]"""
import json
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import p2p_inputs as G  # noqa: E402
import paper_2511_21535_b200 as P  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c5w"
gs = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "2,4,8").split(",")]
inp = G.plummer_tiles(12_500_000, 256, 1, 0) if wl == "c5w" else G.config(wl)
N = inp.pos.shape[0]
for nr in gs:
    grp = P.p2p_loopback_group_create(nr)
    comms = [P.p2p_comm_create_loopback(grp, r) for r in range(nr)]
    bounds = np.linspace(0, N, nr + 1).astype(np.int64)
    res, errs = [None] * nr, []

    def rank_main(r):
        try:
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                sl = slice(bounds[r], bounds[r + 1])
                pos = torch.from_numpy(np.ascontiguousarray(inp.pos[sl])).cuda()
                m = torch.from_numpy(np.ascontiguousarray(inp.mass[sl])).cuda()
                plan = P.Plan(P.P2P_GRAVITY, pos, m, inp.h, inp.lo, inp.nbox, inp.periodic, eps=inp.eps,
                              stream=stream, comm=comms[r])
                i = plan.info
                res[r] = (int(i.n_pairs), int(i.n_local), int(i.n_red))
                plan.close()
        except Exception as e:  # noqa: BLE001
            errs.append((r, repr(e)))

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(nr)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for c in comms:
        P.p2p_comm_destroy(c)
    P.p2p_loopback_group_destroy(grp)
    if errs:
        print(json.dumps({"G": nr, "errors": errs}), flush=True)
        continue
    I = np.array([x[0] for x in res], float)
    n = np.array([x[1] for x in res], float)
    print(json.dumps({"workload": wl, "G": nr, "pairs_per_rank": I.tolist(), "local_particles": n.tolist(),
                      "pairs_max_over_mean": I.max() / I.mean(), "particles_max_over_mean": n.max() / n.mean(),
                      "splitters": os.environ.get("P2P_SPLIT_COST", "count")}), flush=True)
