"""Quick check of the tensor-core Helmholtz path against the CUDA-core kernel and the oracle on c2a/c2b-like
inputs (small first).  usage: python scripts/helm_tc_check.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import p2p_inputs as G  # noqa: E402
import paper_2511_21535_b200 as P  # noqa: E402

for n, t in [(8, 16), (8, 64), (37, 16), (64, 64)]:
    inp = G.dbim_lattice(n, t, seed=3)
    xr = torch.from_numpy(inp.x.view(np.float32).reshape(-1, 2)).cuda()
    with P.Plan(P.P2P_HELMHOLTZ2D, torch.from_numpy(inp.pos).cuda(), xr, inp.h, inp.lo, inp.nbox, 0, k=inp.k,
                t=inp.t) as plan:
        plan.restructure()
        y = plan.eval(P.P2P_REDUNDANT).cpu().numpy()
        yi = plan.eval(P.P2P_INDEXED).cpu().numpy()
    yc = y[:, 0] + 1j * y[:, 1]
    yic = yi[:, 0] + 1j * yi[:, 1]
    ref = oracle.HelmholtzPlan(inp).eval_table()
    msg = f"n={n} t={t}: rel(TC vs indexed SIMT) {oracle.rel_l2(yc, yic):.3e}"
    if ref is not None:
        msg += f"  rel(TC vs oracle) {oracle.rel_l2(yc, ref):.3e}  rel(SIMT vs oracle) {oracle.rel_l2(yic, ref):.3e}"
    print(msg, flush=True)
