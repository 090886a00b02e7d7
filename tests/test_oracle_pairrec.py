"""Pins of the oracle's pair-record mode (the paper's thread-level redundancy, P:L338;
S:L113-116 RedundantBuffers; partial results + deterministic update) against things other
than itself: closed-form record volumes, the symmetry of the neighbour relation, the independently built
box-level redundant buffer (every record is two of its segments, bit for bit), the list-free O(N^2) brute force,
two-body and worked-example closed forms.  CPU only."""
import json
import math
import os

import numpy as np
import pytest

import oracle
import p2p_inputs as G

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _single(pos, mass, eps=1e-3, n=4, dtype=np.float64):
    return G.GravityInput(np.ascontiguousarray(np.asarray(pos, dtype=dtype)),
                          np.ascontiguousarray(np.asarray(mass, dtype=dtype)), (0.0, 0.0, 0.0), 1.0 / n,
                          (n, n, n), 0b111, eps)


def test_c1_record_volume_closed_form():
    # C1: 64 boxes x 27 neighbours, 16 per box: each record holds 16 targets + 16 sources
    gp = oracle.GravityPlan(G.config("c1"))
    off, pr = gp.build_pairrec()
    assert gp.n_nbr == 64 * 27
    assert int(off[-1]) == 64 * 27 * 32 == 55_296 == 2 * gp.R
    assert np.all(np.diff(off.astype(np.int64)) == 32)
    assert pr.shape == (55_296, 4)


@pytest.mark.parametrize("seed", range(4))
def test_target_volume_equals_R_by_symmetry(seed):
    # sum_b |N(b)| n_b == sum_b sum_{k in N(b)} n_k = R because k in N(b) <=> b in N(k), on ragged
    # random inputs with periodic, open and mixed boundaries; records = targets + sources = 2 R
    rng = np.random.default_rng(300 + seed)
    per = [0b111, 0, 0b010, 0b101][seed]
    nbox = tuple(int(v) for v in rng.integers(3, 7, size=3))
    inp = G.random_gravity(int(rng.integers(50, 500)), 0, seed=seed, dtype=np.float64, periodic=per, nbox=nbox,
                           h=0.17, lo=(-0.3, 0.2, 1.0))
    gp = oracle.GravityPlan(inp)
    off, _ = gp.build_pairrec(records=False)
    nb = np.diff(gp.bstart.astype(np.int64))
    T = int((np.diff(gp.nbr_off.astype(np.int64)) * nb).sum())
    assert T == gp.R
    assert int(off[-1]) == T + gp.R


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_records_are_red_segments(dtype):
    """every pair record = [b's own (slot-13) segment of red ; entry e's segment of red], bit for bit, against
    the independently built box-level redundant buffer (orc_gravity_red)"""
    inp = G.plummer(3000, 6, seed=4, dtype=dtype)
    gp = oracle.GravityPlan(inp)
    off, pr = gp.build_pairrec()
    red = gp.red
    nb = np.diff(gp.bstart.astype(np.int64))
    for b in range(gp.B):
        e0, e1 = int(gp.nbr_off[b]), int(gp.nbr_off[b + 1])
        seg = [int(gp.red_off[b])]
        for e in range(e0, e1):
            seg.append(seg[-1] + int(nb[gp.nbr_box[e]]))
        self_e = e0 + int(np.nonzero(gp.nbr_slot[e0:e1] == 13)[0][0])
        own = red[seg[self_e - e0]:seg[self_e - e0 + 1]]
        for e in range(e0, e1):
            r = int(off[e])
            assert pr[r:r + nb[b]].tobytes() == own.tobytes()
            assert pr[r + nb[b]:int(off[e + 1])].tobytes() == red[seg[e - e0]:seg[e - e0 + 1]].tobytes()


@pytest.mark.parametrize("seed", range(5))
def test_pairrec_matches_brute_force(seed):
    """pair-record partials + update vs the list-free O(N^2) brute force (mode iii), fp64: 1e-13"""
    rng = np.random.default_rng(400 + seed)
    per = [0b111, 0, 0b011, 0b100, 0b111][seed]
    nbox = tuple(int(v) for v in rng.integers(3, 6, size=3))
    inp = G.random_gravity(int(rng.integers(40, 400)), 0, seed=seed, dtype=np.float64, periodic=per, nbox=nbox,
                           h=0.2, lo=(0.1, -0.4, 0.0))
    gp = oracle.GravityPlan(inp)
    phi, field, partial = gp.eval_pairrec()
    ref_phi, ref_f = oracle.gravity_brute(inp)
    assert oracle.rel_l2(phi, ref_phi) < 1e-13
    assert oracle.rel_l2(field, ref_f) < 1e-13
    assert partial.shape[0] == gp.R


def test_pairrec_two_body_and_wrap_closed_forms():
    # two bodies in neighbouring boxes: phi = -m/sqrt(d^2+eps^2), |a| = m d/(d^2+eps^2)^{3/2}
    eps = 1e-3
    inp = _single([[0.45, 0.5, 0.5], [0.55, 0.5, 0.5]], [1.0, 1.0], eps=eps)
    dd = inp.pos[1, 0] - inp.pos[0, 0]
    phi, field, _ = oracle.GravityPlan(inp).eval_pairrec()
    assert phi[0] == pytest.approx(-1.0 / math.sqrt(dd * dd + eps * eps), rel=1e-14)
    assert field[0, 0] == pytest.approx(dd / (dd * dd + eps * eps) ** 1.5, rel=1e-14)
    assert field[1, 0] == pytest.approx(-field[0, 0], rel=1e-15)
    # the periodic wrap through the box-level image, stored golden values
    gold = json.load(open(os.path.join(GOLD, "gravity_worked_examples.json")))["ex1_wrap"]
    f32 = lambda v: float(np.float32(v))
    inp = _single([[f32(0.01), 0.5, 0.5], [f32(0.99), 0.5, 0.5]], [1.0, 1.0])
    phi, field, _ = oracle.GravityPlan(inp).eval_pairrec()
    assert phi[0] == pytest.approx(gold["phi_A"], rel=1e-13) and phi[1] == pytest.approx(gold["phi_A"], rel=1e-13)
    assert field[0, 0] == pytest.approx(gold["ax_A"], rel=1e-13)


def test_pairrec_lattice_centres_closed_form():
    # one particle per box at the centres, periodic: a = 0, phi = -m[6/sqrt(h^2+e^2)+12/sqrt(2h^2+e^2)+8/sqrt(3h^2+e^2)]
    n, eps = 4, 1e-3
    h = 1.0 / n
    g = (np.arange(n) + 0.5) * h
    pos = np.array([[x, y, z] for z in g for y in g for x in g])
    phi, field, partial = oracle.GravityPlan(_single(pos, np.ones(len(pos)), eps=eps, n=n)).eval_pairrec()
    ref = -(6 / math.sqrt(h * h + eps * eps) + 12 / math.sqrt(2 * h * h + eps * eps) + 8 / math.sqrt(3 * h * h + eps * eps))
    assert np.allclose(phi, ref, rtol=1e-13, atol=0)
    assert np.max(np.abs(field)) < 1e-12
    assert partial.shape == (64 * 27, 4)


def test_fp32_pairrec_within_rounding():
    # fp32 records: within fp32 rounding of the plain definition (mode ii)
    gp = oracle.GravityPlan(G.config("c1"))
    p1, f1, _ = gp.eval_pairrec()
    p2, f2 = gp.eval_indexed()
    assert oracle.rel_l2(p1, p2) < 1e-6 and oracle.rel_l2(f1, f2) < 1e-6
