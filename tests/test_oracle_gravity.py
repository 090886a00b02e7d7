"""Pins of the gravity oracle (oracle/p2p_oracle.c) against things other than itself:
hand-computed Morton keys, face/boundary binning cases, numpy's stable argsort, O(B^2) box-adjacency
brute force, closed-form counts, closed-form potentials, mpmath worked examples, Newton's third law,
and the oracle's list-free O(N^2) brute force (mode iii).  CPU only."""
import json
import math
import os

import numpy as np
import pytest

import oracle
import p2p_inputs as G

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------------------------------------- a1
def test_morton_hand_values():
    # SURVEY §8c pins: key(1,0,0)=1, (0,1,0)=2, (0,0,1)=4, (1,1,1)=7, (2,0,0)=8, (3,3,3)=63
    for c, k in [((1, 0, 0), 1), ((0, 1, 0), 2), ((0, 0, 1), 4), ((1, 1, 1), 7), ((2, 0, 0), 8), ((3, 3, 3), 63)]:
        assert oracle.morton(3, 2, c) == k
        assert oracle.demorton(3, 2, k) == c
    assert oracle.morton(2, 2, (1, 0)) == 1 and oracle.morton(2, 2, (0, 1)) == 2 and oracle.morton(2, 2, (3, 3)) == 15


def _magic_bits_morton3(x, y, z):
    """an independent 'magic numbers' formulation of the 3D interleave (10 bits per dim)"""
    def spread(v):
        v &= 0x3FF
        v = (v | (v << 16)) & 0x030000FF
        v = (v | (v << 8)) & 0x0300F00F
        v = (v | (v << 4)) & 0x030C30C3
        v = (v | (v << 2)) & 0x09249249
        return v
    return spread(x) | (spread(y) << 1) | (spread(z) << 2)


def test_morton_matches_magic_bits():
    rng = np.random.default_rng(3)
    for _ in range(300):
        c = [int(v) for v in rng.integers(0, 1024, size=3)]
        assert oracle.morton(3, 10, c) == _magic_bits_morton3(*c)


def test_bits_per_dim():
    assert oracle.bits_per_dim((4, 4, 4)) == 2
    assert oracle.bits_per_dim((108, 108, 108)) == 7
    assert oracle.bits_per_dim((512, 256, 256)) == 9
    assert oracle.bits_per_dim((1, 1, 1)) == 0


def test_binning_faces_and_domain():
    # points exactly on box faces land in the upper box; x = lo + n h is out of domain (C6)
    ib = oracle.bin_positions([[0.25, 0.5, 0.0]], 0.25, (0, 0, 0), (4, 4, 4))
    assert tuple(ib[0]) == (1, 2, 0)
    with pytest.raises(oracle.OutOfDomain):
        oracle.bin_positions([[1.0, 0.5, 0.5]], 0.25, (0, 0, 0), (4, 4, 4))
    with pytest.raises(oracle.OutOfDomain):
        oracle.bin_positions([[-1e-9, 0.5, 0.5]], 0.25, (0, 0, 0), (4, 4, 4))
    with pytest.raises(oracle.OutOfDomain):
        oracle.bin_positions([[float("nan"), 0.5, 0.5]], 0.25, (0, 0, 0), (4, 4, 4))
    # shifted origin
    ib = oracle.bin_positions([[-0.74, 10.01, 0.0]], 0.5, (-1.0, 10.0, -0.5), (4, 4, 4))
    assert tuple(ib[0]) == (0, 0, 1)


# ---------------------------------------------------------------------------------------------- a2
def test_stable_sort_matches_numpy():
    rng = np.random.default_rng(1)
    for n in [0, 1, 7, 1000]:
        key = rng.integers(0, 17, size=n).astype(np.uint32)   # many ties
        skey, perm = oracle.stable_sort(key)
        ref = np.argsort(key, kind="stable")
        assert np.array_equal(perm, ref.astype(np.uint32))
        assert np.array_equal(skey, key[ref])


# ------------------------------------------------------------------------------------------ a4, a5
def _brute_adjacency(gp, inp):
    """O(B^2) all-box-pairs adjacency with explicit periodic wrap, independent of the CSR code."""
    nb = oracle.bits_per_dim(inp.nbox)
    coords = np.array([oracle.demorton(3, nb, int(k)) for k in gp.bkey])
    nbox = np.array(inp.nbox)
    out = []
    for b in range(gp.B):
        lst = []
        for k in range(gp.B):
            d = coords[k] - coords[b]
            slot = []
            ok = True
            for q in range(3):
                v = d[q]
                if (inp.periodic >> q) & 1:
                    v = ((v + 1) % nbox[q]) - 1
                if v < -1 or v > 1:
                    ok = False
                slot.append(v)
            if ok:
                lst.append((9 * (slot[2] + 1) + 3 * (slot[1] + 1) + (slot[0] + 1), k))
        out.append(sorted(lst))
    return out


@pytest.mark.parametrize("case", ["c1", "ragged_open", "ragged_mixed"])
def test_neighbour_csr_brute_force(case):
    if case == "c1":
        inp = G.config("c1")
    elif case == "ragged_open":
        inp = G.random_gravity(300, 5, seed=4, periodic=0)
    else:
        inp = G.random_gravity(300, 0, seed=5, periodic=0b101, nbox=(3, 4, 5), h=0.2)
    gp = oracle.GravityPlan(inp, with_red=False)
    ref = _brute_adjacency(gp, inp)
    for b in range(gp.B):
        got = [(int(gp.nbr_slot[e]), int(gp.nbr_box[e])) for e in range(gp.nbr_off[b], gp.nbr_off[b + 1])]
        assert got == ref[b]
    # symmetry b in N(a) <=> a in N(b)
    pairs = {(b, int(gp.nbr_box[e])) for b in range(gp.B) for e in range(gp.nbr_off[b], gp.nbr_off[b + 1])}
    assert all((k, b) in pairs for (b, k) in pairs)


def test_c1_counts_closed_form():
    inp = G.config("c1")
    gp = oracle.GravityPlan(inp)
    assert gp.B == 64 and gp.n_nbr == 64 * 27
    assert gp.R == 27 * 1024 and gp.I == 1024 * 27 * 16      # R = 27N when every box is full and periodic
    counts = np.diff(gp.bstart.astype(np.int64))
    assert counts.sum() == inp.n and np.all(counts == 16)
    # box keys ascending and the box of every sorted particle is its run
    assert np.all(np.diff(gp.bkey.astype(np.int64)) > 0)


def test_red_round_trip_multiset():
    """every record of box b's run, shifted back by its slot image and origin, is a source particle of a
    box adjacent to b (by brute force), each such particle exactly once (S:L156 round trip)."""
    inp = G.random_gravity(400, 4, seed=9, dtype=np.float64)
    gp = oracle.GravityPlan(inp)
    pos = inp.pos
    ib = oracle.bin_positions(pos, inp.h, inp.lo, inp.nbox)
    for b in range(gp.B):
        i0 = gp.perm[gp.bstart[b]]
        cb = ib[i0]
        adj = []
        for j in range(inp.n):
            d = (ib[j] - cb + 1) % 4 - 1
            if np.all(np.abs(d) <= 1):
                adj.append(j)
        run = gp.red[gp.red_off[b]:gp.red_off[b + 1]]
        assert len(run) == len(adj)
        assert np.array_equal(np.sort(run[:, 3]), np.sort(inp.mass[adj]))
        # local coordinates lie inside the 3-box neighbourhood of the target box origin
        assert np.all(run[:, :3] >= -inp.h - 1e-12) and np.all(run[:, :3] < 2 * inp.h + 1e-12)


# ---------------------------------------------------------------------------------------------- a7
def _single(pos, mass, eps=1e-3, n=4, dtype=np.float32):
    return G.GravityInput(np.ascontiguousarray(np.asarray(pos, dtype=dtype)),
                          np.ascontiguousarray(np.asarray(mass, dtype=dtype)), (0.0, 0.0, 0.0), 1.0 / n,
                          (n, n, n), 0b111, eps)


def _all_modes(inp):
    """modes (ii) and (iii) are exact in fp64; mode (i) evaluates on the working-precision rebased
    records, so for fp32 inputs it is only within fp32 rounding -- callers use _exact_modes for tight
    pins and check mode (i) separately."""
    gp = oracle.GravityPlan(inp)
    return [gp.eval_indexed(), gp.eval_redundant(), oracle.gravity_brute(inp)]


def _exact_modes(inp):
    gp = oracle.GravityPlan(inp)
    return [gp.eval_indexed(), oracle.gravity_brute(inp)]


def test_two_body_closed_form():
    # |a| = m d / (d^2+eps^2)^{3/2}, phi = -m / sqrt(d^2+eps^2)  (S:L205 with eps > 0)
    d, eps = 0.1, 1e-3
    inp = _single([[0.45, 0.5, 0.5], [0.55, 0.5, 0.5]], [1.0, 1.0], eps=eps, n=4, dtype=np.float64)
    dd = inp.pos[1, 0] - inp.pos[0, 0]
    for phi, field in _all_modes(inp):
        assert phi[0] == pytest.approx(-1.0 / math.sqrt(dd * dd + eps * eps), rel=1e-14)
        assert field[0, 0] == pytest.approx(dd / (dd * dd + eps * eps) ** 1.5, rel=1e-14)
        assert field[1, 0] == pytest.approx(-field[0, 0], rel=1e-15)
        assert abs(field[0, 1]) < 1e-300 and abs(field[0, 2]) < 1e-300


def test_spec_unit_force():
    # two unit masses at distance 1 -> force magnitude 1, opposite directions (eps -> 0)
    inp = G.GravityInput(np.array([[0.5, 0.5, 0.5], [1.5, 0.5, 0.5]]), np.array([1.0, 1.0]), (0.0, 0.0, 0.0), 1.0,
                         (3, 3, 3), 0, 1e-9)
    for phi, field in _all_modes(inp):
        assert field[0, 0] == pytest.approx(1.0, rel=1e-12) and field[1, 0] == pytest.approx(-1.0, rel=1e-12)


def test_collinear_triple_middle_zero():
    # three equal collinear equally spaced particles -> middle net force 0
    inp = _single([[0.3, 0.5, 0.5], [0.4, 0.5, 0.5], [0.5, 0.5, 0.5]], [1.0, 1.0, 1.0], n=2 ** 2, dtype=np.float64)
    inp.pos[:, 0] = [0.375 - 0.0625, 0.375, 0.375 + 0.0625]     # exact binary spacing
    for phi, field in _all_modes(inp):
        assert np.all(np.abs(field[1]) <= 1e-12 * np.abs(field[0, 0]))


def test_lattice_centres_closed_form():
    # one particle per box at the box centres, periodic, equal masses: a = 0 by symmetry and
    # phi = -m[6/sqrt(h^2+e^2) + 12/sqrt(2h^2+e^2) + 8/sqrt(3h^2+e^2)]  (SURVEY §8c derived closed form)
    gold = json.load(open(os.path.join(GOLD, "gravity_worked_examples.json")))["lattice_centres"]
    for n in [4, 5]:
        h, eps = 1.0 / n, 1e-3
        g = (np.arange(n) + 0.5) * h
        pos = np.array([[x, y, z] for z in g for y in g for x in g])
        inp = _single(pos, np.ones(len(pos)), eps=eps, n=n, dtype=np.float64)
        ref = -(6 / math.sqrt(h * h + eps * eps) + 12 / math.sqrt(2 * h * h + eps * eps) + 8 / math.sqrt(3 * h * h + eps * eps))
        if n == 4:
            assert ref == pytest.approx(gold["phi"], rel=1e-14)
        for phi, field in _all_modes(inp):
            assert np.allclose(phi, ref, rtol=1e-13, atol=0)
            assert np.max(np.abs(field)) < 1e-12


def test_worked_examples_mpmath():
    """SURVEY §8c Ex1 (wrap), Ex2 (direct neighbour), Ex3 (box rule, not distance), re-derived live with
    mpmath and compared with the stored SURVEY values."""
    mp = pytest.importorskip("mpmath")
    mp.mp.dps = 30
    gold = json.load(open(os.path.join(GOLD, "gravity_worked_examples.json")))
    eps = 1e-3
    f32 = lambda v: float(np.float32(v))
    xa, xb, xc, xd = f32(0.01), f32(0.99), f32(0.49), f32(0.51)

    def pair(d):
        d = mp.mpf(d)
        r2 = d * d + mp.mpf(eps) ** 2
        return float(-1 / mp.sqrt(r2)), float(d / r2 ** mp.mpf(1.5))

    # Ex1: A (box 0) and B (box 3) interact through the image B - 1
    dA = (mp.mpf(xb) - 1) - mp.mpf(xa)
    assert float(dA) == pytest.approx(gold["ex1_wrap"]["d_A"], rel=1e-15)
    phiA, axA = pair(dA)
    assert phiA == pytest.approx(gold["ex1_wrap"]["phi_A"], rel=1e-14)
    assert axA == pytest.approx(gold["ex1_wrap"]["ax_A"], rel=1e-14)
    inp = _single([[xa, 0.5, 0.5], [xb, 0.5, 0.5]], [1.0, 1.0])
    for phi, field in _exact_modes(inp):
        assert phi[0] == pytest.approx(phiA, rel=1e-13) and phi[1] == pytest.approx(phiA, rel=1e-13)
        assert field[0, 0] == pytest.approx(axA, rel=1e-13) and field[1, 0] == pytest.approx(-axA, rel=1e-13)
    phi, field = oracle.GravityPlan(inp).eval_redundant()       # fp32 rebased records: fp32 rounding only
    assert phi[0] == pytest.approx(phiA, rel=1e-5) and field[1, 0] == pytest.approx(-axA, rel=1e-5)
    # Ex2: A (box 0) and C (box 1) direct neighbours
    phiC, axC = pair(mp.mpf(xc) - mp.mpf(xa))
    assert phiC == pytest.approx(gold["ex2_direct"]["phi_contrib"], rel=1e-14)
    assert axC == pytest.approx(gold["ex2_direct"]["ax_contrib_on_A"], rel=1e-14)
    inp = _single([[xa, 0.5, 0.5], [xc, 0.5, 0.5]], [1.0, 1.0])
    for phi, field in _exact_modes(inp):
        assert phi[0] == pytest.approx(phiC, rel=1e-13) and field[0, 0] == pytest.approx(axC, rel=1e-13)
    # Ex3: A (box 0) and D (box 2) are not neighbours for n = 4 although |d| < h*2.1
    inp = _single([[xa, 0.5, 0.5], [xd, 0.5, 0.5]], [1.0, 1.0])
    for phi, field in _all_modes(inp):
        assert phi[0] == 0.0 and np.all(field == 0.0)


@pytest.mark.parametrize("seed", range(6))
def test_modes_agree_with_brute_force(seed):
    """oracle modes (i) redundant order and (ii) indexed order vs the list-free O(N^2) brute force (iii),
    on ragged random inputs with periodic, open and mixed boundaries (fp64: 1e-13)."""
    rng = np.random.default_rng(100 + seed)
    per = [0b111, 0, 0b010, 0b101, 0b111, 0b111][seed]
    nbox = tuple(int(v) for v in rng.integers(3, 7, size=3))
    inp = G.random_gravity(int(rng.integers(50, 600)), 0, seed=seed, dtype=np.float64, periodic=per, nbox=nbox,
                           h=0.17, lo=(-0.3, 0.2, 1.0))
    gp = oracle.GravityPlan(inp)
    ref_phi, ref_f = oracle.gravity_brute(inp)
    for phi, field in (gp.eval_indexed(), gp.eval_redundant()):
        assert oracle.rel_l2(phi, ref_phi) < 1e-13
        assert oracle.rel_l2(field, ref_f) < 1e-13


def test_fp32_redundant_order_within_rounding():
    # fp32 records hold fl32 rebased coordinates; mode (i) on them stays within fp32 rounding of (ii)
    inp = G.config("c1")
    gp = oracle.GravityPlan(inp)
    (p1, f1), (p2, f2) = gp.eval_redundant(), gp.eval_indexed()
    assert oracle.rel_l2(p1, p2) < 1e-6 and oracle.rel_l2(f1, f2) < 1e-6


def test_newton_third_law():
    # sum_i m_i a_i = 0 for the symmetric kernel over a symmetric pair list
    for inp in [G.uniform_per_box(6, 8, seed=2, dtype=np.float64), G.plummer(4000, 8, seed=3, dtype=np.float64)]:
        gp = oracle.GravityPlan(inp)
        _, field = gp.eval_indexed()
        ma = inp.mass[:, None] * field
        assert np.max(np.abs(ma.sum(axis=0))) <= 1e-12 * np.abs(ma).sum()


def test_empty_and_single():
    inp = _single(np.zeros((0, 3)), np.zeros(0), dtype=np.float64)
    gp = oracle.GravityPlan(inp)
    assert gp.B == 0 and gp.R == 0
    inp = _single([[0.1, 0.2, 0.3]], [2.0], dtype=np.float64)
    for phi, field in _all_modes(inp):
        assert phi[0] == 0.0 and np.all(field == 0.0)


@pytest.mark.parametrize("dt,per", [(np.float64, 0b111), (np.float32, 0b101), (np.float64, 0b000)])
def test_red_round_trip_coordinates_nonzero_lo(dt, per):
    """C11 pinned from outside with lo != 0: every record of box b's run, moved back by b's
    origin lo + c_b h (computed here from the box key by plain arithmetic, not by the oracle's fma), is its source
    particle (identified by its unique mass) up to ONE periodic image S_d in {-L_d, 0, +L_d} (0 if open), that
    image is the box-level one (the source box, shifted by S, is a stencil neighbour of b), and the record lies
    in [-h, 2h) of b's origin.  A wrong origin, a wrong image sign or a transposed component fails here."""
    lo, h, nbox = (-0.4, 0.25, 2.0), 0.13, (5, 4, 6)
    inp = G.random_gravity(1500, 0, seed=31, dtype=dt, periodic=per, nbox=nbox, h=h, lo=lo)
    assert len(np.unique(inp.mass)) == inp.n
    gp = oracle.GravityPlan(inp)
    nb = oracle.bits_per_dim(nbox)
    ib = oracle.bin_positions(inp.pos, h, lo, nbox)
    L = np.array(nbox, np.float64) * h
    by_mass = {float(m): j for j, m in enumerate(inp.mass)}
    ulp = np.finfo(dt).eps
    for b in range(gp.B):
        cb = np.array(oracle.demorton(3, nb, int(gp.bkey[b])), np.float64)
        o = np.array(lo) + cb * h
        run = gp.red[gp.red_off[b]:gp.red_off[b + 1]].astype(np.float64)
        for rec in run:
            j = by_mass[float(dt(rec[3]))]
            S = rec[:3] + o - inp.pos[j].astype(np.float64)
            img = np.rint(S / L)
            assert np.all(np.abs(S - img * L) <= 8 * ulp * (np.abs(o) + 2 * h + L))
            for d in range(3):
                assert img[d] in (-1, 0, 1) and (img[d] == 0 or (per >> d) & 1)
            delta = ib[j] + img * np.array(nbox) - cb
            assert np.all(np.abs(delta) <= 1)
            assert np.all(rec[:3] >= -h * (1 + 1e-6)) and np.all(rec[:3] < 2 * h * (1 + 1e-6))
