"""Multi-PROCESS path: G separate OS processes (one per rank, all on the one B200
the tests reach -- NCCL refuses several ranks per device, so they talk through p2p_comm_create_ipc: CUDA IPC peer
memory + a shared-memory barrier) run the whole collective algorithm: supercell histogram all-reduce, device
splitters, one all-to-all-v routing owners + halo, local plan, reverse all-to-all-v of the results, and a second
collective time step (p2p_plan_update).  Every rank's outputs for its own slice must equal BIT FOR BIT the 1-GPU
plan over the rank-major concatenation, and the oracle within the stated tolerance."""
import os
import secrets
import subprocess
import sys

import numpy as np
import pytest

import oracle
import p2p_bounds as bounds
import p2p_inputs as G

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2511_21535_b200 as P
    return P


def single(P, pos, mass, inp):
    out = {}
    with P.Plan(P.P2P_GRAVITY, torch.from_numpy(pos).cuda(), torch.from_numpy(mass).cuda(), inp.h, inp.lo, inp.nbox,
                inp.periodic, eps=inp.eps) as plan:
        plan.restructure()
        for lay in ("redundant", "indexed", "indexed_bitwise"):
            phi, f = plan.eval(P.LAYOUTS[lay])
            out[lay] = (phi.cpu().numpy(), f.cpu().numpy())
    return out


@pytest.mark.parametrize("nr,case", [(2, "plummer"), (3, "plummer"), (4, "uniform")])
def test_multiprocess_ipc_bitwise_equals_single_gpu(P, tmp_path, nr, case):
    if case == "plummer":
        inp = G.plummer(30000, 16, seed=40 + nr)
    else:
        inp = G.uniform_per_box(12, 6, seed=40 + nr)
    rng = np.random.default_rng(nr)
    cuts = np.sort(rng.choice(np.arange(1, inp.n), nr - 1, replace=False))
    cuts = np.concatenate([[0], cuts, [inp.n]])
    # step 2: every particle moved a little (re-wrapped into the periodic domain, kept below the upper face)
    L = np.asarray(inp.nbox) * inp.h
    pos2 = (inp.pos.astype(np.float64) + rng.normal(0, 0.3 * inp.h, inp.pos.shape)) % L
    pos2 = np.minimum(pos2, L * (1 - 1e-7)).astype(inp.pos.dtype)
    path = str(tmp_path / "inp.npz")
    np.savez(path, pos=inp.pos, mass=inp.mass, pos2=pos2, h=inp.h, lo=np.asarray(inp.lo), nbox=np.asarray(inp.nbox),
             periodic=inp.periodic, eps=inp.eps, cuts=cuts)
    name = "p2ptest_" + secrets.token_hex(8)
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "mp_rank.py"), str(r), str(nr), name, path,
                               str(tmp_path)], stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(nr)]
    logs = []
    for p in procs:
        try:
            o, _ = p.communicate(timeout=600)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            pytest.fail("a rank process hung")
        logs.append(o)
    assert all(p.returncode == 0 for p in procs), "\n".join(logs)
    ref = single(P, inp.pos, inp.mass, inp)
    ref2 = single(P, pos2, inp.mass, inp)
    gp = oracle.GravityPlan(inp)
    rphi, rf = gp.eval_indexed()
    for r in range(nr):
        d = np.load(str(tmp_path / f"rank{r}.npz"))
        sl = slice(int(cuts[r]), int(cuts[r + 1]))
        for lay in ("redundant", "indexed", "indexed_bitwise"):
            assert d[f"{lay}_phi"].tobytes() == ref[lay][0][sl].tobytes(), (r, lay)
            assert d[f"{lay}_field"].tobytes() == ref[lay][1][sl].tobytes(), (r, lay)
        assert d["step2_phi"].tobytes() == ref2["redundant"][0][sl].tobytes(), r
        assert d["step2_field"].tobytes() == ref2["redundant"][1][sl].tobytes(), r
        assert bounds.close(d["redundant_phi"], rphi[sl], 1e-5) and bounds.close(d["redundant_field"], rf[sl], 1e-5)
    # every rank derived the same splitters on its device
    sp = [tuple(np.load(str(tmp_path / f"rank{r}.npz"))["splitters"]) for r in range(nr)]
    assert len(set(sp)) == 1


def test_ipc_name_collision_rejected(P):
    """rank 0 refuses an existing rendezvous name (stale segment / concurrent group)"""
    name = "p2ptest_" + secrets.token_hex(8)
    path = "/dev/shm/" + name
    open(path, "wb").close()
    try:
        with pytest.raises(P.P2PError) as e:
            P.p2p_comm_create_ipc(2, 0, name)
        assert e.value.status == P.P2P_ERR_INVALID_ARGUMENT
    finally:
        os.unlink(path)
