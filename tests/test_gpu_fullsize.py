"""Full-size parity at BASELINE.json's sizes, in the configuration bench.py times (-m gpu):

* gravity c5w (configs[4] per-GPU tile: 12.5M Plummer particles, 256^3 periodic boxes), built through the same
  persistent-plan p2p_plan_update path the bench step uses: sorted keys, permutation, box table, neighbour CSR
  and red_off compared with the oracle over the WHOLE input; the redundant buffer compared byte for byte on
  sampled boxes; potentials / fields of every target of 400 seeded-random boxes (plus the densest boxes) against
  the fp64 oracle (plain definition) -- relative L2 <= 1e-5 over the sample;
* gravity c4-8 (configs[3], 10M particles, the density sweep's hardest point): same sampled checks;
* Helmholtz c2b (configs[1]: 256^2 leaf cells x t = 64): structures over the whole input, y on sampled boxes.
"""
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


def _sample_boxes(gp, n, seed):
    rng = np.random.default_rng(seed)
    nb = np.diff(gp.bstart.astype(np.int64))
    dense = np.argsort(nb)[-20:]                       # the densest boxes (longest runs, several work items)
    pick = rng.choice(gp.B, size=min(n, gp.B), replace=False)
    return np.unique(np.concatenate([pick, dense]))


def _check_gravity(P, inp, seed):
    gp = oracle.GravityPlan(inp, with_red=False)
    pos = torch.from_numpy(inp.pos).cuda()
    m = torch.from_numpy(inp.mass).cuda()
    # the bench's configuration: one persistent plan, each step an asynchronous p2p_plan_update
    plan = P.Plan(P.P2P_GRAVITY, pos, m, inp.h, inp.lo, inp.nbox, inp.periodic, eps=inp.eps)
    try:
        plan.update(pos, m)
        plan.restructure()
        phi, f = plan.eval(P.P2P_REDUNDANT)
        phi_i, f_i = plan.eval(P.P2P_INDEXED)
        torch.cuda.synchronize()
        info = plan.refresh_info()
        assert info.n_boxes == gp.B and info.n_nbr == gp.n_nbr and info.n_red == gp.R and info.n_pairs == gp.I
        assert np.array_equal(plan.copy_out(P.P2P_ARR_SORTED_KEYS), gp.skey)
        assert np.array_equal(plan.copy_out(P.P2P_ARR_PERM), gp.perm)
        assert np.array_equal(plan.copy_out(P.P2P_ARR_BOX_KEYS), gp.bkey)
        assert np.array_equal(plan.copy_out(P.P2P_ARR_BOX_START), gp.bstart)
        assert np.array_equal(plan.copy_out(P.P2P_ARR_NBR_OFF), gp.nbr_off)
        assert np.array_equal(plan.copy_out(P.P2P_ARR_NBR_BOX), gp.nbr_box)
        assert np.array_equal(plan.copy_out(P.P2P_ARR_NBR_SLOT), gp.nbr_slot)
        assert np.array_equal(plan.copy_out(P.P2P_ARR_RED_OFF), gp.red_off)
        boxes = _sample_boxes(gp, 400, seed)
        # red[] on the sampled boxes' runs, byte for byte against the oracle's records
        red = plan.copy_out(P.P2P_ARR_RED)
        ref_red = _oracle_red_runs(gp, boxes)
        for b, run in ref_red.items():
            assert red[gp.red_off[b]:gp.red_off[b + 1]].tobytes() == run.tobytes(), b
    finally:
        plan.close()
    rphi, rf = gp.eval_indexed_boxes(boxes)
    sel = np.concatenate([gp.perm[gp.bstart[b]:gp.bstart[b + 1]] for b in boxes])
    for (gphi, gf) in ((phi.cpu().numpy(), f.cpu().numpy()), (phi_i.cpu().numpy(), f_i.cpu().numpy())):
        assert bounds.close(gphi[sel], rphi[sel], 1e-5)
        assert bounds.close(gf[sel], rf[sel], 1e-5)
    return len(sel)


def _oracle_red_runs(gp, boxes):
    """the oracle's redundant records of the listed boxes only (a sub-plan over the same structures)"""
    sub = oracle.GravityPlan.__new__(oracle.GravityPlan)
    sub.__dict__.update(gp.__dict__)
    out = {}
    for b in boxes:
        # a one-box view: red_off rebased to 0 for box b
        view = dict(bkey=gp.bkey[b:b + 1], nbr_off=(gp.nbr_off[b:b + 2] - gp.nbr_off[b]).astype(np.uint32),
                    nbr_box=gp.nbr_box[gp.nbr_off[b]:gp.nbr_off[b + 1]],
                    nbr_slot=gp.nbr_slot[gp.nbr_off[b]:gp.nbr_off[b + 1]],
                    red_off=(gp.red_off[b:b + 2] - gp.red_off[b]).astype(np.uint64))
        sub.__dict__.update(view)
        sub.B = 1
        sub.R = int(gp.red_off[b + 1] - gp.red_off[b])
        out[int(b)] = sub.build_red().copy()
    return out


@pytest.mark.timeout(1200)
def test_fullsize_c5w_tile(P):
    assert _check_gravity(P, G.plummer_tiles(12_500_000, 256, 1, 0), seed=1) > 1000


@pytest.mark.timeout(1200)
def test_fullsize_c4_8(P):
    assert _check_gravity(P, G.config("c4-8"), seed=2) > 1000


@pytest.mark.timeout(1200)
def test_fullsize_c2b_helmholtz(P):
    inp = G.config("c2b")
    hp = oracle.HelmholtzPlan(inp)
    xr = torch.from_numpy(inp.x.view(np.float32).reshape(-1, 2)).cuda()
    with P.Plan(P.P2P_HELMHOLTZ2D, torch.from_numpy(inp.pos).cuda(), xr, inp.h, inp.lo, inp.nbox, 0, k=inp.k,
                t=inp.t) as plan:
        assert plan.info.n_boxes == hp.B == 65536 and plan.info.n_pairs == hp.n_pairs
        assert np.array_equal(plan.copy_out(P.P2P_ARR_PERM), hp.perm)
        assert np.array_equal(plan.copy_out(P.P2P_ARR_NBR_BOX), hp.nbr9.ravel())
        plan.restructure()
        y = plan.eval(P.P2P_REDUNDANT).cpu().numpy()
        y = y[:, 0] + 1j * y[:, 1]
    # the oracle on sampled boxes: y_b = P Xg_b from the oracle's own table and im2col
    rng = np.random.default_rng(4)
    boxes = rng.choice(hp.B, 300, replace=False)
    Xg = hp.xg()[boxes].reshape(len(boxes), -1)
    yb = Xg @ hp.P.T
    sel = np.concatenate([hp.perm[hp.bstart[b]:hp.bstart[b + 1]] for b in boxes])
    assert bounds.close(y[sel], yb.ravel(), 1e-5)
