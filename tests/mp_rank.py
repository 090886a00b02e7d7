"""One rank of the multi-PROCESS test (tests/test_gpu_multiproc.py): a separate OS process that joins an IPC
communicator (p2p_comm_create_ipc: CUDA IPC peer memory, all ranks may share one GPU), runs the collective plan on
its input slice -- build, restructure, every layout, then one collective p2p_plan_update time step -- and saves its
outputs.  usage: python tests/mp_rank.py RANK NRANKS NAME INPUT.npz OUTDIR"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_21535_b200 as P  # noqa: E402


def main():
    rank, nr, name, inp_path, outdir = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4], sys.argv[5]
    torch.cuda.set_device(rank % torch.cuda.device_count())
    d = np.load(inp_path)
    cuts = d["cuts"]
    sl = slice(int(cuts[rank]), int(cuts[rank + 1]))
    pos = torch.from_numpy(np.ascontiguousarray(d["pos"][sl])).cuda()
    m = torch.from_numpy(np.ascontiguousarray(d["mass"][sl])).cuda()
    comm = P.p2p_comm_create_ipc(nr, rank, name)
    stream = torch.cuda.Stream()
    res = {}
    with torch.cuda.stream(stream):
        plan = P.Plan(P.P2P_GRAVITY, pos, m, float(d["h"]), tuple(d["lo"]), tuple(int(v) for v in d["nbox"]),
                      int(d["periodic"]), eps=float(d["eps"]), stream=stream, comm=comm)
        res["splitters"] = P.p2p_get_splitters(plan.handle, nr)
        plan.restructure()
        for lay in ("redundant", "indexed", "indexed_bitwise"):
            phi, f = plan.eval(P.LAYOUTS[lay])
            stream.synchronize()
            res[f"{lay}_phi"], res[f"{lay}_field"] = phi.cpu().numpy(), f.cpu().numpy()
        # a second time step with moved particles (the collective update: new partition, new exchange)
        pos2 = torch.from_numpy(np.ascontiguousarray(d["pos2"][sl])).cuda()
        plan.update(pos2, m)
        plan.restructure()
        phi, f = plan.eval(P.P2P_REDUNDANT)
        stream.synchronize()
        res["step2_phi"], res["step2_field"] = phi.cpu().numpy(), f.cpu().numpy()
        plan.close()
    P.p2p_comm_destroy(comm)
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), **res)
    print(f"rank {rank} done", flush=True)


if __name__ == "__main__":
    main()
