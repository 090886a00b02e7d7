"""GPU parity of the pair-record layout (the paper's thread-level redundancy,
P:L338, with per-record partials and the deterministic update) through the C ABI vs the fp64 oracle:
the record buffer bit for bit, potentials and fields within 1e-5 (fp32) / 1e-12 (fp64) of the plain definition
(mode ii), bitwise run-to-run determinism, state errors."""
import numpy as np
import pytest

import oracle
import p2p_bounds as bounds
import p2p_inputs as G

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {np.float32: 1e-5, np.float64: 1e-12}


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2511_21535_b200 as P
    return P


def gpu_plan(P, inp):
    pos = torch.from_numpy(inp.pos).cuda()
    m = torch.from_numpy(inp.mass).cuda()
    return P.Plan(P.P2P_GRAVITY, pos, m, inp.h, inp.lo, inp.nbox, inp.periodic, eps=inp.eps)


CASES = ["c1", "c1_f64", "plummer", "open", "mixed", "big_box"]


def make(case):
    if case == "c1":
        return G.config("c1")
    if case == "c1_f64":
        return G.config("c1", dtype=np.float64)
    if case == "plummer":
        return G.plummer(20000, 12, seed=3)
    if case == "open":
        return G.random_gravity(3000, 0, seed=4, periodic=0, nbox=(7, 5, 6), h=0.15, lo=(-0.2, 0.1, 0.0))
    if case == "mixed":
        return G.random_gravity(4000, 0, seed=5, dtype=np.float64, periodic=0b101, nbox=(5, 4, 6), h=0.2)
    # one box holding 700 particles plus sparse neighbours: several target / source chunks of 32
    rng = np.random.default_rng(6)
    pos = np.concatenate([0.5 + 0.1 * rng.uniform(size=(700, 3)), rng.uniform(size=(300, 3))]).astype(np.float32)
    mass = rng.uniform(0.5, 1.5, size=1000).astype(np.float32) / 1000
    return G.GravityInput(pos, mass, (0.0, 0.0, 0.0), 0.25, (4, 4, 4), 0b111, 1e-3)


@pytest.mark.parametrize("case", CASES)
def test_pairrec_records_and_values(P, case):
    inp = make(case)
    dt = inp.pos.dtype.type
    gp = oracle.GravityPlan(inp)
    off, pr = gp.build_pairrec()
    ref_phi, ref_f = gp.eval_indexed()
    with gpu_plan(P, inp) as plan:
        plan.restructure_pairs()
        nrec, nslot = P.p2p_get_pairrec_size(plan.handle)
        assert nrec == int(off[-1]) and nslot == gp.R          # T = R by neighbour symmetry
        assert plan.copy_out(P.P2P_ARR_PAIRREC).tobytes() == pr.tobytes()
        phi, f = plan.eval(P.P2P_PAIRREC)
        phi2, f2 = plan.eval(P.P2P_PAIRREC)
        torch.cuda.synchronize()
        phi, f, phi2, f2 = (x.cpu().numpy() for x in (phi, f, phi2, f2))
    assert phi.tobytes() == phi2.tobytes() and f.tobytes() == f2.tobytes()   # deterministic update
    assert bounds.close(phi, ref_phi, TOL[dt]), case
    assert bounds.close(f, ref_f, TOL[dt]), case
    if dt == np.float64:   # fp64: also within 1e-12 of the oracle's own pair-record evaluation
        p3, f3, _ = gp.eval_pairrec()
        assert bounds.close(phi, p3, 1e-12) and bounds.close(f, f3, 1e-12)


def test_pairrec_plummer_1e6_sampled(P):
    """BASELINE configs[2] (10^6 Plummer, 128^3 boxes) at full size: the pair-record eval vs the oracle's plain
    definition on a seeded sample of target boxes"""
    inp = G.config("c3")
    gp = oracle.GravityPlan(inp, with_red=False)
    sel = np.sort(np.random.default_rng(7).choice(gp.B, 3000, replace=False))
    rphi, rf = gp.eval_indexed_boxes(sel)
    mask = ~np.isnan(rphi)
    with gpu_plan(P, inp) as plan:
        plan.restructure_pairs()
        phi, f = plan.eval(P.P2P_PAIRREC)
        phi, f = phi.cpu().numpy(), f.cpu().numpy()
    assert bounds.close(phi[mask], rphi[mask], 1e-5)
    assert bounds.close(f[mask], rf[mask], 1e-5)


def test_pairrec_state_errors(P):
    inp = G.config("c1")
    with gpu_plan(P, inp) as plan:
        with pytest.raises(P.P2PError) as e:
            plan.eval(P.P2P_PAIRREC)
        assert e.value.status == P.P2P_ERR_BAD_STATE
        plan.restructure_pairs()
        plan.eval(P.P2P_PAIRREC)
        plan.update(torch.from_numpy(inp.pos).cuda(), torch.from_numpy(inp.mass).cuda())
        with pytest.raises(P.P2PError) as e:
            plan.eval(P.P2P_PAIRREC)
        assert e.value.status == P.P2P_ERR_BAD_STATE
        plan.restructure_pairs()                                   # rebuilt after the update
        phi, _ = plan.eval(P.P2P_PAIRREC)
        ref, _ = oracle.GravityPlan(inp, with_red=False).eval_indexed()
        assert bounds.close(phi.cpu().numpy(), ref, 1e-5)
    h = G.dbim_lattice(4, 4, seed=0)
    xr = torch.from_numpy(h.x.view(np.float32).reshape(-1, 2)).cuda()
    with P.Plan(P.P2P_HELMHOLTZ2D, torch.from_numpy(h.pos).cuda(), xr, h.h, h.lo, h.nbox, 0, k=h.k, t=h.t) as plan:
        with pytest.raises(P.P2PError) as e:
            plan.restructure_pairs()
        assert e.value.status == P.P2P_ERR_UNSUPPORTED
