"""GPU parity of the gravity path (-m gpu): the CUDA library through its C ABI vs the fp64 oracle.

Bars (BASELINE north_star): sort order, box table, neighbour lists and redundant buffers bit-exact; potentials
and fields within relative L2 1e-5 (fp32) / 1e-12 (fp64) of the oracle's plain definition (mode ii);
P2P_REDUNDANT == P2P_INDEXED_BITWISE bit for bit."""
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


def check_structs(P, plan, gp):
    assert plan.info.n_boxes == gp.B and plan.info.n_nbr == gp.n_nbr
    assert plan.info.n_red == gp.R and plan.info.n_pairs == gp.I
    assert np.array_equal(plan.copy_out(P.P2P_ARR_SORTED_KEYS), gp.skey)
    assert np.array_equal(plan.copy_out(P.P2P_ARR_PERM), gp.perm)
    assert np.array_equal(plan.copy_out(P.P2P_ARR_BOX_KEYS), gp.bkey)
    assert np.array_equal(plan.copy_out(P.P2P_ARR_BOX_START), gp.bstart)
    assert np.array_equal(plan.copy_out(P.P2P_ARR_NBR_OFF), gp.nbr_off)
    assert np.array_equal(plan.copy_out(P.P2P_ARR_NBR_BOX), gp.nbr_box)
    assert np.array_equal(plan.copy_out(P.P2P_ARR_NBR_SLOT), gp.nbr_slot)
    assert np.array_equal(plan.copy_out(P.P2P_ARR_RED_OFF), gp.red_off)


def run_all_layouts(P, plan):
    plan.restructure()
    out = {}
    for name, lay in P.LAYOUTS.items():
        phi, f = plan.eval(lay)
        torch.cuda.synchronize()
        out[name] = (phi.cpu().numpy(), f.cpu().numpy())
    return out


def check_case(P, inp, structs=True):
    dt = inp.pos.dtype.type
    gp = oracle.GravityPlan(inp)
    ref_phi, ref_f = gp.eval_indexed()
    with gpu_plan(P, inp) as plan:
        if structs:
            check_structs(P, plan, gp)
        out = run_all_layouts(P, plan)
        if structs:
            red = plan.copy_out(P.P2P_ARR_RED)
            assert red.tobytes() == gp.red.tobytes()     # bit-exact redundant buffer
    for name, (phi, f) in out.items():
        assert bounds.close(phi, ref_phi, TOL[dt]), name
        assert bounds.close(f, ref_f, TOL[dt]), name
    # REDUNDANT and INDEXED_BITWISE stage identical bits -> identical outputs
    assert out["redundant"][0].tobytes() == out["indexed_bitwise"][0].tobytes()
    assert out["redundant"][1].tobytes() == out["indexed_bitwise"][1].tobytes()
    return out


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_c1(P, dtype):
    check_case(P, G.uniform_per_box(4, 16, seed=0, dtype=dtype))


@pytest.mark.parametrize("seed", range(8))
def test_ragged_random_boundaries(P, seed):
    rng = np.random.default_rng(200 + seed)
    per = [0b111, 0, 0b010, 0b101, 0b111, 0b011, 0b111, 0][seed]
    nbox = tuple(int(v) for v in rng.integers(3, 9, size=3))
    dt = np.float64 if seed % 2 else np.float32
    inp = G.random_gravity(int(rng.integers(100, 3000)), 0, seed=seed, dtype=dt, periodic=per, nbox=nbox, h=0.13,
                           lo=(-0.4, 0.25, 2.0))
    check_case(P, inp)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_plummer_clustered(P, dtype):
    # dense clustered boxes: > 128 targets per box (several work items), runs longer than one pipeline stage
    check_case(P, G.plummer(20000, 8, seed=1, dtype=dtype))


def test_hundred_c1_scenarios(P):
    """>= 100 seeded C1-sized scenarios (S:L590 acceptance criterion 1), structures + values"""
    for seed in range(100):
        inp = G.uniform_per_box(4, 16, seed=seed) if seed % 2 == 0 else G.random_gravity(1024, 4, seed=seed)
        check_case(P, inp, structs=(seed % 10 == 0))


def test_edge_cases(P):
    # single particle, all particles in one box, one box per dim, empty input
    one = G.GravityInput(np.array([[0.1, 0.2, 0.3]], np.float32), np.array([0.5], np.float32), (0, 0, 0), 0.25,
                         (4, 4, 4), 0b111, 1e-3)
    out = check_case(P, one)
    assert out["redundant"][0][0] == 0.0 and np.all(out["redundant"][1] == 0.0)
    rng = np.random.default_rng(0)
    box = G.GravityInput((0.5 + 0.2 * rng.random((700, 3))).astype(np.float32),
                         rng.uniform(0.5, 1.5, 700).astype(np.float32) / 700, (0, 0, 0), 1.0, (1, 1, 1), 0, 1e-2)
    check_case(P, box)
    empty = G.GravityInput(np.zeros((0, 3), np.float32), np.zeros(0, np.float32), (0, 0, 0), 0.25, (4, 4, 4), 0b111,
                           1e-3)
    with gpu_plan(P, empty) as plan:
        assert plan.info.n_boxes == 0
        plan.restructure()
        phi, f = plan.eval(P.P2P_REDUNDANT)
        assert phi.numel() == 0


def test_errors(P):
    inp = G.uniform_per_box(4, 2, seed=0)
    bad = inp.pos.copy()
    bad[17, 1] = 1.0                     # x = lo + n h is outside the domain (C6)
    with pytest.raises(P.P2PError) as e:
        gpu_plan(P, G.GravityInput(bad, inp.mass, inp.lo, inp.h, inp.nbox, inp.periodic, inp.eps))
    assert e.value.status == P.P2P_ERR_OUT_OF_DOMAIN and "17" in str(e.value)
    with gpu_plan(P, inp) as plan:
        with pytest.raises(P.P2PError) as e:
            plan.eval(P.P2P_REDUNDANT)   # before restructure
        assert e.value.status == P.P2P_ERR_BAD_STATE
        plan.restructure()
        plan.eval(P.P2P_REDUNDANT)
        plan.set_charges(torch.from_numpy(inp.mass * 2).cuda())
        with pytest.raises(P.P2PError) as e:
            plan.eval(P.P2P_REDUNDANT)   # red[] invalidated by set_charges
        assert e.value.status == P.P2P_ERR_BAD_STATE
    # host pointers rejected
    cfg = P.make_config(P.P2P_GRAVITY, P.P2P_FP32, inp.h, inp.lo, inp.nbox, inp.periodic, eps=1e-3)
    with pytest.raises(P.P2PError) as e:
        P.p2p_plan_create(cfg, inp.n, inp.pos.ctypes.data, inp.mass.ctypes.data)
    assert e.value.status == P.P2P_ERR_INVALID_ARGUMENT


def test_set_charges_reuses_geometry(P):
    inp = G.uniform_per_box(5, 8, seed=3)
    m2 = (inp.mass * np.float32(1.7)).astype(np.float32)
    ref = oracle.GravityPlan(G.GravityInput(inp.pos, m2, inp.lo, inp.h, inp.nbox, inp.periodic, inp.eps))
    rphi, rf = ref.eval_indexed()
    with gpu_plan(P, inp) as plan:
        plan.set_charges(torch.from_numpy(m2).cuda())
        plan.restructure()
        for lay in P.LAYOUTS.values():
            phi, f = plan.eval(lay)
            assert bounds.close(phi.cpu().numpy(), rphi, 1e-5)
            assert bounds.close(f.cpu().numpy(), rf, 1e-5)


def test_determinism(P):
    inp = G.plummer(30000, 16, seed=7)
    res = []
    for _ in range(2):
        with gpu_plan(P, inp) as plan:
            res.append(run_all_layouts(P, plan))
    for name in res[0]:
        assert res[0][name][0].tobytes() == res[1][name][0].tobytes()
        assert res[0][name][1].tobytes() == res[1][name][1].tobytes()


def test_nearfield_host_api(P):
    inp = G.uniform_per_box(6, 8, seed=11)
    phi, f = P.nearfield(P.P2P_GRAVITY, torch.from_numpy(inp.pos), torch.from_numpy(inp.mass), inp.h, inp.lo,
                         inp.nbox, inp.periodic, eps=inp.eps)
    assert not phi.is_cuda
    rphi, rf = oracle.GravityPlan(inp).eval_indexed()
    assert bounds.close(phi.numpy(), rphi, 1e-5) and bounds.close(f.numpy(), rf, 1e-5)


def test_plan_update_time_steps(P):
    """p2p_plan_update: asynchronous rebuild for moved particles (PhotoNs time step); N may shrink or grow;
    structures and values equal a fresh oracle build of the new input"""
    a = G.plummer(5000, 6, seed=1)
    seq = [G.plummer(4000, 6, seed=2), G.uniform_per_box(6, 8, seed=3), G.plummer(9000, 6, seed=4)]
    with gpu_plan(P, a) as plan:
        for inp in seq:
            plan.update(torch.from_numpy(inp.pos).cuda(), torch.from_numpy(inp.mass).cuda())
            plan.restructure()
            phi, f = plan.eval(P.P2P_REDUNDANT)
            gp = oracle.GravityPlan(inp)
            check_structs(P, plan, gp)
            assert plan.copy_out(P.P2P_ARR_RED).tobytes() == gp.red.tobytes()
            rphi, rf = gp.eval_indexed()
            assert bounds.close(phi.cpu().numpy(), rphi, 1e-5) and bounds.close(f.cpu().numpy(), rf, 1e-5)
            phi2, f2 = plan.eval(P.P2P_INDEXED)
            assert bounds.close(phi2.cpu().numpy(), rphi, 1e-5) and bounds.close(f2.cpu().numpy(), rf, 1e-5)


def test_plan_update_reports_out_of_domain(P):
    inp = G.uniform_per_box(4, 4, seed=0)
    bad = inp.pos.copy()
    bad[5, 2] = -0.01
    with gpu_plan(P, inp) as plan:
        plan.update(torch.from_numpy(bad).cuda(), torch.from_numpy(inp.mass).cuda())   # asynchronous: no error yet
        with pytest.raises(P.P2PError) as e:
            plan.refresh_info()
        assert e.value.status == P.P2P_ERR_OUT_OF_DOMAIN and "5" in str(e.value)
        plan.update(torch.from_numpy(inp.pos).cuda(), torch.from_numpy(inp.mass).cuda())
        assert plan.refresh_info().n_boxes == 64


def test_host_buffer_entry_points(P):
    """p2p_plan_update_host / p2p_eval_host (the bench's e2e path): the library's own H2D / D2H copies give the
    same bits as the device entry points, and the values match the oracle"""
    a = G.plummer(6000, 6, seed=21)
    seq = [G.plummer(7000, 6, seed=22), G.uniform_per_box(6, 5, seed=23)]   # same geometry as a
    with gpu_plan(P, a) as plan:
        for inp in seq:
            pos_h = torch.from_numpy(inp.pos).pin_memory()
            m_h = torch.from_numpy(inp.mass).pin_memory()
            plan.update_host(pos_h, m_h)
            plan.restructure()
            phi_h, f_h = plan.eval_host(P.P2P_REDUNDANT)
            assert not phi_h.is_cuda and not f_h.is_cuda
            plan.update(pos_h.cuda(), m_h.cuda())
            plan.restructure()
            phi_d, f_d = plan.eval(P.P2P_REDUNDANT)
            torch.cuda.synchronize()
            assert phi_h.numpy().tobytes() == phi_d.cpu().numpy().tobytes()
            assert f_h.numpy().tobytes() == f_d.cpu().numpy().tobytes()
            rphi, rf = oracle.GravityPlan(inp).eval_indexed()
            assert bounds.close(phi_h.numpy(), rphi, 1e-5) and bounds.close(f_h.numpy(), rf, 1e-5)
            # numpy inputs (pageable) work too; device pointers are rejected
            plan.update_host(inp.pos, inp.mass)
            plan.restructure()
            phi2, _ = plan.eval_host(P.P2P_REDUNDANT, want_field=False)
            assert phi2.numpy().tobytes() == phi_h.numpy().tobytes()
        with pytest.raises(P.P2PError) as e:
            P.p2p_eval_host(plan.handle, P.P2P_REDUNDANT, phi_d.data_ptr(), None)
        assert e.value.status == P.P2P_ERR_INVALID_ARGUMENT
