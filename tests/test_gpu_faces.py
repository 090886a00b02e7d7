"""GPU parity on box faces: positions exactly on interior faces lo + k h, one ulp either side
of them, just below the upper face lo + n h, with negative and non-representable lo.  C6 bins with one fp64 IEEE
division of the promoted position and rejects computed indices outside [0, n): the GPU must make the SAME decision
for every such point -- sorted keys, permutation, box table, CSR and red[] byte-equal to the oracle, and a point
the oracle rejects rejected by the GPU with the same index.  Random inputs never hit faces; these do."""
import numpy as np
import pytest

import oracle
import p2p_inputs as G
import p2p_bounds as bounds

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GEOMS = [  # (lo, h, nbox, periodic)
    ((0.0, 0.0, 0.0), 0.25, (4, 4, 4), 0b111),
    ((-0.4, 0.25, 2.0), 0.13, (5, 6, 7), 0b101),
    ((-1000.3, 7.77, -3.1), 0.37, (4, 5, 6), 0b111),
    ((0.1, -0.7, 0.3), 0.1, (3, 9, 4), 0b000),
]


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2511_21535_b200 as P
    return P


def _face_candidates(lo, h, n, dt):
    """working-precision values at and around every face lo + k h, k = 0..n (the nearest value and its two
    neighbours), plus the largest value below the upper face"""
    out = []
    for k in range(n + 1):
        f = dt(np.float64(lo) + np.float64(k) * np.float64(h))
        out += [np.nextafter(f, dt(-np.inf)), f, np.nextafter(f, dt(np.inf))]
    return np.array(out, dt)


def _accepted(v, lo, h, n):
    """which candidate values the ORACLE bins inside [0, n) along one dimension"""
    ok = np.zeros(len(v), bool)
    for i, x in enumerate(v):
        try:
            oracle.bin_positions(np.array([[x, lo[1], lo[2]]]), h, lo, (n, 1 << 20, 1 << 20))
            ok[i] = True
        except oracle.OutOfDomain:
            pass
    return ok


def face_input(geom, dt, seed, n_pts=3000):
    lo, h, nbox, per = geom
    rng = np.random.default_rng(seed)
    cols, rejected = [], []
    for d in range(3):
        lo_d = tuple(lo[d] if e == 0 else lo[e] for e in range(3))
        cand = _face_candidates(lo[d], h, nbox[d], dt)
        acc = _accepted(cand.astype(np.float64), (lo[d], lo[1], lo[2]), h, nbox[d])
        rejected.append(cand[~acc])
        good = cand[acc]
        rand = (lo[d] + nbox[d] * h * rng.uniform(1e-6, 1 - 1e-6, n_pts)).astype(dt)
        pick = rng.random(n_pts) < 0.6                      # 60% of the coordinates on / next to a face
        cols.append(np.where(pick, good[rng.integers(0, len(good), n_pts)], rand))
    pos = np.ascontiguousarray(np.stack(cols, axis=1).astype(dt))
    m = (rng.uniform(0.5, 1.5, n_pts) / n_pts).astype(dt)
    return G.GravityInput(pos, m, lo, h, nbox, per, 1e-3 * h), rejected


def _plan(P, inp):
    return P.Plan(P.P2P_GRAVITY, torch.from_numpy(inp.pos).cuda(), torch.from_numpy(inp.mass).cuda(), inp.h,
                  inp.lo, inp.nbox, inp.periodic, eps=inp.eps)


@pytest.mark.parametrize("gi", range(len(GEOMS)))
@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_faces_bit_exact(P, gi, dt):
    inp, _ = face_input(GEOMS[gi], dt, seed=10 + gi)
    gp = oracle.GravityPlan(inp)
    tol = 1e-5 if dt == np.float32 else 1e-12
    rphi, rf = gp.eval_indexed()
    with _plan(P, inp) as plan:
        assert plan.info.n_boxes == gp.B and plan.info.n_red == gp.R and plan.info.n_pairs == gp.I
        for arr, ref in [(P.P2P_ARR_SORTED_KEYS, gp.skey), (P.P2P_ARR_PERM, gp.perm), (P.P2P_ARR_BOX_KEYS, gp.bkey),
                         (P.P2P_ARR_BOX_START, gp.bstart), (P.P2P_ARR_NBR_OFF, gp.nbr_off),
                         (P.P2P_ARR_NBR_BOX, gp.nbr_box), (P.P2P_ARR_NBR_SLOT, gp.nbr_slot),
                         (P.P2P_ARR_RED_OFF, gp.red_off)]:
            assert np.array_equal(plan.copy_out(arr), ref), arr
        plan.restructure()
        assert plan.copy_out(P.P2P_ARR_RED).tobytes() == gp.red.tobytes()
        for lay in P.LAYOUTS.values():
            phi, f = plan.eval(lay)
            assert bounds.close(phi.cpu().numpy(), rphi, tol) and bounds.close(f.cpu().numpy(), rf, tol), lay


@pytest.mark.parametrize("gi", range(len(GEOMS)))
@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_faces_rejections_agree(P, gi, dt):
    """every candidate the oracle rejects (computed index outside [0, n)) is rejected by the GPU at its index"""
    inp, rejected = face_input(GEOMS[gi], dt, seed=20 + gi, n_pts=200)
    n_checked = 0
    for d in range(3):
        for x in rejected[d]:
            pos = inp.pos.copy()
            pos[137, d] = x
            bad = G.GravityInput(pos, inp.mass, inp.lo, inp.h, inp.nbox, inp.periodic, inp.eps)
            with pytest.raises(oracle.OutOfDomain):
                oracle.GravityPlan(bad, with_red=False)
            with pytest.raises(P.P2PError) as e:
                _plan(P, bad)
            assert e.value.status == P.P2P_ERR_OUT_OF_DOMAIN and "137" in str(e.value)
            n_checked += 1
    assert n_checked >= 6      # at least lo - ulp and lo + n h per dimension
