"""Multi-GPU path on one GPU: G emulated ranks (host threads sharing the device, loopback
communicators) run the full collective algorithm -- supercell histogram all-reduce, count-balanced Morton
splitters (computed on the device), one all-to-all-v routing every particle to its owner and as a halo source to
every other rank owning one of its box's neighbours, local plan over the received records, reverse all-to-all-v of
the results.  Each rank's outputs for its own input slice must equal, BIT FOR BIT, the 1-GPU plan over the rank-major
concatenation of the slices (SURVEY §8e "bitwise identical to 1 GPU"), and match the fp64 oracle."""
import threading

import numpy as np
import pytest

import oracle
import p2p_bounds as bounds
import p2p_inputs as G

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2511_21535_b200 as P
    return P


def run_ranks(P, inp, slices, layouts):
    """one thread per emulated rank; returns per-rank {layout: (phi, field)} and per-rank info"""
    nr = len(slices)
    grp = P.p2p_loopback_group_create(nr)
    comms = [P.p2p_comm_create_loopback(grp, r) for r in range(nr)]
    out = [None] * nr
    infos = [None] * nr
    errs = []

    def rank_main(r):
        try:
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                sl = slices[r]
                pos = torch.from_numpy(np.ascontiguousarray(inp.pos[sl])).cuda()
                m = torch.from_numpy(np.ascontiguousarray(inp.mass[sl])).cuda()
                plan = P.Plan(P.P2P_GRAVITY, pos, m, inp.h, inp.lo, inp.nbox, inp.periodic, eps=inp.eps,
                              stream=stream, comm=comms[r])
                infos[r] = (plan.info, P.p2p_get_splitters(plan.handle, nr))
                plan.restructure()
                res = {}
                for lay in layouts:
                    phi, f = plan.eval(lay)
                    stream.synchronize()
                    res[lay] = (phi.cpu().numpy(), f.cpu().numpy())
                out[r] = res
                plan.close()
        except Exception as e:  # noqa: BLE001 -- surfaced below
            errs.append((r, e))

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(nr)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    for c in comms:
        P.p2p_comm_destroy(c)
    P.p2p_loopback_group_destroy(grp)
    assert not errs, errs
    return out, infos


def single(P, inp, layouts):
    pos = torch.from_numpy(inp.pos).cuda()
    m = torch.from_numpy(inp.mass).cuda()
    with P.Plan(P.P2P_GRAVITY, pos, m, inp.h, inp.lo, inp.nbox, inp.periodic, eps=inp.eps) as plan:
        plan.restructure()
        res = {}
        for lay in layouts:
            phi, f = plan.eval(lay)
            res[lay] = (phi.cpu().numpy(), f.cpu().numpy())
        return res, plan.info


def expected_splitters(P, cat, key_bits, nr):
    """p2p_partition_splitters (host) of the global supercell histogram built from the oracle's keys"""
    sc_bits = max(0, min(key_bits - 2, 18))  # supercells >= 4 keys (k_dist.cu)
    shift = key_bits - sc_bits
    hist = np.bincount(oracle.GravityPlan(cat, with_red=False).key >> shift, minlength=1 << sc_bits)
    return P.p2p_partition_splitters(hist.astype(np.uint64), shift, key_bits, nr)


@pytest.mark.parametrize("case", ["plummer_g2", "plummer_g3", "uniform_g4", "open_g2", "skewed_g4", "fp64_g2",
                                  "plummer64_g8", "plummer128_g5", "uniform_g7", "clump_g6"])
def test_multirank_bitwise_equals_single_gpu(P, case):
    rng = np.random.default_rng(17)
    if case.startswith("plummer"):
        inp = G.plummer(30000, 16, seed=5)
    elif case == "uniform_g4":
        inp = G.uniform_per_box(8, 8, seed=6)
    elif case == "open_g2":
        inp = G.random_gravity(5000, 0, seed=7, periodic=0, nbox=(7, 5, 6), h=0.15, lo=(-0.2, 0.1, 0.0))
    elif case == "fp64_g2":
        inp = G.plummer(8000, 8, seed=8, dtype=np.float64)
    elif case == "plummer64_g8":
        inp = G.plummer(60000, 64, seed=10)     # 18-bit keys: one supercell per box
    elif case == "plummer128_g5":
        inp = G.plummer(40000, 128, seed=11)    # 21-bit keys: supercells of 8 boxes
    elif case == "uniform_g7":
        inp = G.uniform_per_box(12, 2, seed=12)
    elif case == "clump_g6":   # one box holds 90% of the particles: several splitters fall in one supercell
        r2 = np.random.default_rng(13)
        pts = np.concatenate([r2.random((400, 3)), 0.52 + 0.1 * r2.random((3600, 3))]).astype(np.float32)
        inp = G.GravityInput(pts, (0.5 + r2.random(4000)).astype(np.float32) / 4000, (0.0, 0.0, 0.0), 0.125,
                             (8, 8, 8), 0b111, 1e-3)
    else:
        inp = G.plummer(20000, 16, seed=9)
    nr = int(case[-1])
    # rank slices: a random (non-spatial) split of uneven sizes; skewed: everything on one rank but one
    perm = rng.permutation(inp.n)
    if case == "skewed_g4":
        cuts = [0, inp.n - 3, inp.n - 2, inp.n - 1, inp.n]
    else:
        cuts = [0] + sorted(rng.choice(np.arange(1, inp.n), nr - 1, replace=False).tolist()) + [inp.n]
    slices = [np.sort(perm[cuts[r]:cuts[r + 1]]) for r in range(nr)]
    concat = np.concatenate(slices)
    cat = G.GravityInput(np.ascontiguousarray(inp.pos[concat]), np.ascontiguousarray(inp.mass[concat]), inp.lo, inp.h,
                         inp.nbox, inp.periodic, inp.eps)
    lays = [P.P2P_REDUNDANT, P.P2P_INDEXED, P.P2P_INDEXED_BITWISE]
    ref, rinfo = single(P, cat, lays)
    out, infos = run_ranks(P, cat, [np.arange(cuts[r], cuts[r + 1]) for r in range(nr)], lays)
    # every target box is owned by exactly one rank: pair counts add up to the 1-GPU plan's
    assert sum(i.n_pairs for i, _ in infos) == rinfo.n_pairs
    # the device-side splitters (k_splitters) equal the host function on the same global histogram, on every rank
    want = expected_splitters(P, cat, rinfo.key_bits, nr)
    for _, spl in infos:
        assert np.array_equal(spl, want), (spl, want)
    for lay in lays:
        phi = np.concatenate([out[r][lay][0] for r in range(nr)])
        fld = np.concatenate([out[r][lay][1] for r in range(nr)])
        assert phi.tobytes() == ref[lay][0].tobytes(), lay
        assert fld.tobytes() == ref[lay][1].tobytes(), lay
    tol = 1e-12 if inp.pos.dtype == np.float64 else 1e-5
    rphi, rf = oracle.GravityPlan(cat, with_red=False).eval_indexed()
    phi = np.concatenate([out[r][P.P2P_REDUNDANT][0] for r in range(nr)])
    assert bounds.close(phi, rphi, tol)


def test_nccl_communicator_single_rank(P):
    """the NCCL backend itself (1 rank on the box's one GPU: all-reduce, grouped send/recv to self)"""
    inp = G.plummer(20000, 16, seed=21)
    uid = P.p2p_comm_unique_id()
    comm = P.p2p_comm_create(1, 0, uid)
    try:
        pos = torch.from_numpy(inp.pos).cuda()
        m = torch.from_numpy(inp.mass).cuda()
        with P.Plan(P.P2P_GRAVITY, pos, m, inp.h, inp.lo, inp.nbox, inp.periodic, eps=inp.eps, comm=comm) as plan:
            plan.restructure()
            phi, f = plan.eval(P.P2P_REDUNDANT)
            phi, f = phi.cpu().numpy(), f.cpu().numpy()
    finally:
        P.p2p_comm_destroy(comm)
    ref, _ = single(P, inp, [P.P2P_REDUNDANT])
    assert phi.tobytes() == ref[P.P2P_REDUNDANT][0].tobytes()
    assert f.tobytes() == ref[P.P2P_REDUNDANT][1].tobytes()


def test_multirank_rank_with_no_particles(P):
    inp = G.uniform_per_box(4, 4, seed=3)
    out, infos = run_ranks(P, inp, [np.arange(inp.n), np.arange(0)], [P.P2P_REDUNDANT])
    ref, _ = single(P, inp, [P.P2P_REDUNDANT])
    assert out[0][P.P2P_REDUNDANT][0].tobytes() == ref[P.P2P_REDUNDANT][0].tobytes()
    assert out[1][P.P2P_REDUNDANT][0].size == 0


@pytest.mark.parametrize("nr", [2, 3])
def test_multirank_plan_update_time_steps(P, nr):
    """p2p_plan_update on a collective plan (a new time step on every rank, the partition recomputed, the plan's
    buffers reused; N per rank changes between steps): bitwise equal to a 1-GPU plan of each step's input"""
    steps = [G.plummer(9000, 8, seed=31), G.plummer(12000, 8, seed=32), G.uniform_per_box(8, 3, seed=33)]
    lay = P.P2P_REDUNDANT
    grp = P.p2p_loopback_group_create(nr)
    comms = [P.p2p_comm_create_loopback(grp, r) for r in range(nr)]
    rng = np.random.default_rng(5)
    cuts = []
    for inp in steps:
        c = np.sort(rng.choice(np.arange(1, inp.n), size=nr - 1, replace=False))
        cuts.append([0, *c.tolist(), inp.n])
    out = [[None] * nr for _ in steps]
    errs = []

    def rank_main(r):
        try:
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                plan = None
                for k, inp in enumerate(steps):
                    sl = slice(cuts[k][r], cuts[k][r + 1])
                    pos = torch.from_numpy(np.ascontiguousarray(inp.pos[sl])).cuda()
                    m = torch.from_numpy(np.ascontiguousarray(inp.mass[sl])).cuda()
                    if plan is None:
                        plan = P.Plan(P.P2P_GRAVITY, pos, m, inp.h, inp.lo, inp.nbox, inp.periodic, eps=inp.eps,
                                      stream=stream, comm=comms[r])
                    else:
                        plan.update(pos, m)
                    plan.restructure()
                    phi, f = plan.eval(lay)
                    stream.synchronize()
                    out[k][r] = (phi.cpu().numpy(), f.cpu().numpy())
                plan.close()
        except Exception as e:  # noqa: BLE001 -- surfaced below
            errs.append((r, e))

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(nr)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    for c in comms:
        P.p2p_comm_destroy(c)
    P.p2p_loopback_group_destroy(grp)
    assert not errs, errs
    for k, inp in enumerate(steps):
        ref, _ = single(P, inp, [lay])
        phi = np.concatenate([out[k][r][0] for r in range(nr)])
        f = np.concatenate([out[k][r][1] for r in range(nr)])
        assert phi.tobytes() == ref[lay][0].tobytes(), k
        assert f.tobytes() == ref[lay][1].tobytes(), k
