"""Multi-box work items of the REDUNDANT eval (k_structs.cu mb_quad, k_eval_gravity.cu MBK): aligned quads of 4
consecutive target boxes with <= 8 targets and <= 65535 sources each are ONE work item whose 4 runs are staged in
lockstep.  Checked: the values against the oracle (plain definition, mode ii, and the redundant-order mode i),
REDUNDANT == INDEXED_BITWISE bit for bit (BITWISE evaluates quad members with the quad's 4 source splits), and
INDEXED within tolerance -- on inputs where every box, some boxes, or no box forms quads."""
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


def mixed_counts(n, seed, dtype=np.float32):
    """per-box counts 3..8 with ~1/4 of the boxes at 9..20 (breaking some quads) and a few empty boxes"""
    rng = np.random.default_rng(seed)
    nb = rng.integers(3, 9, n ** 3)
    big = rng.random(n ** 3) < 0.25
    nb[big] = rng.integers(9, 21, big.sum())
    nb[rng.random(n ** 3) < 0.03] = 0
    cells = np.repeat(np.arange(n ** 3), nb)
    iz, rem = np.divmod(cells, n * n)
    iy, ix = np.divmod(rem, n)
    h = 1.0 / n
    u = rng.uniform(1e-4, 1 - 1e-4, (cells.size, 3))
    pos = np.stack([(ix + u[:, 0]) * h, (iy + u[:, 1]) * h, (iz + u[:, 2]) * h], 1)
    p = rng.permutation(cells.size)
    mass = rng.uniform(0.5, 1.5, cells.size) / cells.size
    return G.GravityInput(np.ascontiguousarray(pos[p].astype(dtype)), np.ascontiguousarray(mass[p].astype(dtype)),
                          (0.0, 0.0, 0.0), h, (n, n, n), 0b111, 1e-3, "mixed")


CASES = {
    "all_quads_8": lambda dt: G.uniform_per_box(10, 8, seed=3, dtype=dt),    # every box: 8 targets, R = 216
    "all_quads_5": lambda dt: G.uniform_per_box(11, 5, seed=4, dtype=dt),    # 5 targets, R = 135 (> SMALL_R)
    "mixed": lambda dt: mixed_counts(12, 5, dt),
    "plummer": lambda dt: G.plummer(40000, 24, seed=6, dtype=dt),
}


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_mbquad_values_and_bitwise(P, case, dt):
    inp = CASES[case](dt)
    gp = oracle.GravityPlan(inp)
    rphi, rf = gp.eval_indexed()
    iphi, if_ = gp.eval_redundant()
    tol = 1e-5 if dt == np.float32 else 1e-12
    with P.Plan(P.P2P_GRAVITY, torch.from_numpy(inp.pos).cuda(), torch.from_numpy(inp.mass).cuda(), inp.h, inp.lo,
                inp.nbox, inp.periodic, eps=inp.eps) as plan:
        plan.restructure()
        red = [t.cpu().numpy() for t in plan.eval(P.P2P_REDUNDANT)]
        bit = [t.cpu().numpy() for t in plan.eval(P.P2P_INDEXED_BITWISE)]
        idx = [t.cpu().numpy() for t in plan.eval(P.P2P_INDEXED)]
        red2 = [t.cpu().numpy() for t in plan.eval(P.P2P_REDUNDANT)]
    assert red[0].tobytes() == bit[0].tobytes() and red[1].tobytes() == bit[1].tobytes()
    assert red[0].tobytes() == red2[0].tobytes() and red[1].tobytes() == red2[1].tobytes()  # deterministic
    assert bounds.close(red[0], rphi, tol) and bounds.close(red[1], rf, tol)
    assert bounds.close(red[0], iphi, tol) and bounds.close(red[1], if_, tol)
    assert bounds.close(idx[0], rphi, tol) and bounds.close(idx[1], rf, tol)
