"""Pins of the adaptive-leaf oracle (oracle/adaptive.py; readings C22-C24 in DESIGN §3).

What fixes it from outside itself:
* leaves: every leaf holds <= t particles unless it is a finest cell; the leaves' runs partition the sorted
  particles; the leaf count equals an independent bottom-up recount (SPEC S:L59's "independent recursive-count
  oracle"); SPEC's trivial examples;
* equal-size leaves reduce to the uniform grid: the closed lists are exactly the 27-stencil CSR of the pinned grid
  oracle (C4, C5 image convention), the redundant records equal its C11 records box by box, and the potentials /
  fields agree with its plain definition;
* the lists are symmetric and equal the range construction the GPU will use; the closure is needed
  (the dilation alone is asymmetric on clustered inputs);
* the eval equals an all-pairs brute force that evaluates the adjacency predicate from the leaf boxes directly
  (no lists), and conserves momentum (Newton's third law, which only the closed pair set guarantees)."""
import numpy as np
import pytest

import oracle
import p2p_inputs as G
from oracle import adaptive as A


def test_spec_trivial_examples():
    # 10 particles, t = 16 -> one leaf; 4 particles at distinct corners, t = 1 -> 4 leaves
    rng = np.random.default_rng(0)
    pts = (0.1 + 0.8 * rng.random((10, 3))).astype(np.float64)
    inp = G.GravityInput(pts, np.ones(10), (0.0, 0.0, 0.0), 1 / 16, (16, 16, 16), 0b111, 1e-3)
    t = A.AdaptiveTree(inp, 16, min_bits=0)
    assert t.nleaf == 1 and t.leaves[0][:2] == (0, 0) and t.leaves[0][3] == 10
    corners = np.array([[0.01, 0.01, 0.01], [0.99, 0.01, 0.01], [0.01, 0.99, 0.99], [0.99, 0.99, 0.99]])
    inp = G.GravityInput(corners, np.ones(4), (0.0, 0.0, 0.0), 1 / 16, (16, 16, 16), 0b111, 1e-3)
    assert A.AdaptiveTree(inp, 1, min_bits=0).nleaf == 4


@pytest.mark.parametrize("t", [1, 4, 16, 64])
def test_leaves_threshold_partition_recount(t):
    inp = G.plummer(4000, 32, seed=3, dtype=np.float64)
    tr = A.AdaptiveTree(inp, t)
    starts = [s for _, _, s, _ in tr.leaves]
    counts = [c for _, _, _, c in tr.leaves]
    assert starts[0] == 0 and all(s + c == s2 for s, c, s2 in zip(starts, counts, starts[1:]))
    assert starts[-1] + counts[-1] == 4000 and min(counts) >= 1
    for (l, _, _, c) in tr.leaves:
        assert c <= t or l == 3 * tr.m
        assert l >= tr.min_bits
    # every particle's key carries its leaf's prefix
    for a, (l, p, s, c) in enumerate(tr.leaves):
        assert np.all(tr.skey[s:s + c] >> (3 * tr.m - l) == p)
    assert tr.nleaf == A.leaf_count_bottom_up(tr.key, tr.m, t, tr.min_bits)


def test_equal_leaves_reduce_to_the_grid_stencil():
    inp = G.uniform_per_box(8, 4, seed=5, dtype=np.float64)          # 8^3 boxes, 4 each; t = 4 -> finest leaves
    tr = A.AdaptiveTree(inp, 4)
    gp = oracle.GravityPlan(inp)
    assert tr.nleaf == gp.B == 512
    n = 8
    nbr = tr.neighbours()
    for b in range(gp.B):
        c = np.array(oracle.demorton(3, 3, int(gp.bkey[b])))
        want = set()
        for e in range(gp.nbr_off[b], gp.nbr_off[b + 1]):
            s = int(gp.nbr_slot[e])
            v = c + np.array([s % 3 - 1, s // 3 % 3 - 1, s // 9 - 1])
            img = np.where(v >= n, 1, np.where(v < 0, -1, 0))          # C5: +L past the upper face
            want.add((int(gp.nbr_box[e]), int(9 * (img[2] + 1) + 3 * (img[1] + 1) + (img[0] + 1))))
        assert set(nbr[b]) == want and len(nbr[b]) == 27
    # C24 records = C11 records, box by box (as multisets: the two list orders differ)
    red = tr.red(np.float64)
    off = 0
    for b in range(gp.B):
        k = int(gp.red_off[b + 1] - gp.red_off[b])
        mine = red[off:off + k]
        ref = gp.red[gp.red_off[b]:gp.red_off[b + 1]]
        assert np.array_equal(mine[np.lexsort(mine.T[::-1])], ref[np.lexsort(ref.T[::-1])])
        off += k
    phi, f = tr.eval(inp.eps)
    rphi, rf = gp.eval_indexed()
    assert oracle.rel_l2(phi, rphi) <= 1e-13 and oracle.rel_l2(f, rf) <= 1e-13


@pytest.mark.parametrize("seed,t", [(1, 8), (2, 16), (4, 3)])
def test_symmetry_closure_and_range_construction(seed, t):
    inp = G.plummer(3000, 32, seed=seed, dtype=np.float64)
    tr = A.AdaptiveTree(inp, t)
    nbr = tr.neighbours()
    sets = [set(x) for x in nbr]
    for a in range(tr.nleaf):
        assert (a, 13) in sets[a]                                       # self, no image
        for b, code in nbr[a]:
            assert (a, 26 - code) in sets[b]
    assert tr.neighbours_by_ranges() == nbr
    # the closure is not a formality: the dilation alone is asymmetric on clustered leaves
    ov = tr._overlap0()
    assert (ov != ov[:, ::-1, :].transpose(2, 1, 0)).any()


def test_eval_equals_brute_force_and_conserves_momentum():
    inp = G.plummer(1500, 16, seed=7, dtype=np.float64)
    tr = A.AdaptiveTree(inp, 6)
    phi, f = tr.eval(inp.eps)
    bphi, bf = A.brute(tr, inp.eps)
    assert oracle.rel_l2(phi, bphi) <= 1e-12 and oracle.rel_l2(f, bf) <= 1e-12
    mom = (tr.mass[:, None] * f).sum(axis=0)
    assert np.abs(mom).max() <= 1e-12 * np.abs(tr.mass[:, None] * f).sum()
    # interaction count (C19: i = j included) = the acting (i, j, S) triples of the predicate + the N self pairs
    assert tr.pair_count() == A.brute_pairs(tr) + len(tr.key)


def test_single_leaf_lists_and_eval_match_the_all_pairs_ones():
    # the per-leaf forms used for full-size sampled checks equal the all-pairs definition
    inp = G.plummer(2500, 32, seed=9, dtype=np.float64)
    tr = A.AdaptiveTree(inp, 8)
    nbr = tr.neighbours()
    phi, f = tr.eval(inp.eps)
    for a in range(0, tr.nleaf, 37):
        assert A.neighbours_of(tr, a) == nbr[a]
        ti, p, ff = A.eval_leaf(tr, a, inp.eps)
        assert np.allclose(p, phi[ti], rtol=1e-14, atol=0) and np.allclose(ff, f[ti], rtol=1e-13, atol=1e-300)


@pytest.mark.parametrize("seed,t,lo", [(11, 3, (-0.3, 0.7, 1.1)), (12, 8, (0.0, 0.0, 0.0)), (13, 20, (2.5, -1.25, 0.6))])
def test_red_round_trip_unequal_leaves(seed, t, lo):
    """C24 pinned from outside for UNEQUAL leaves and lo != 0 (value checks cannot catch a wrong
    origin because it cancels in d = s - t): for every target leaf a, with a's origin and width recomputed here
    from its (level, prefix) pair by plain arithmetic, every record of a's run moved back by that origin and its
    entry's image S is its source particle (unique mass), the source lies inside leaf b's own cell, the pair is
    adjacent in the closed sense (b + S overlaps a dilated by a's width, or a - S overlaps b dilated by b's), and
    dilation entries (b no coarser than a) lie in [-w_a, 2 w_a) of a's origin."""
    base = G.plummer(2500, 16, seed=seed, dtype=np.float64)
    pos = np.ascontiguousarray(base.pos + np.array(lo))
    inp = G.GravityInput(pos, base.mass, lo, base.h, base.nbox, base.periodic, base.eps)
    assert len(np.unique(inp.mass)) == inp.n
    tr = A.AdaptiveTree(inp, t)
    n = tr.n
    L = float(n * inp.h)
    levels = {l for l, _, _, _ in tr.leaves}
    assert len(levels) >= 3                                   # genuinely unequal leaves
    nbr = tr.neighbours()
    red = tr.red(np.float64)
    by_mass = {float(m): j for j, m in enumerate(inp.mass)}

    def cell(leaf):
        l, p, _, _ = tr.leaves[leaf]
        sx, sy, sz = l // 3, (l + 1) // 3, (l + 2) // 3       # halvings per dimension (z first)
        c = [0, 0, 0]
        key = p << (3 * tr.m - l)                             # the cell's first finest key
        for k in range(tr.m):
            for d in range(3):
                c[d] |= ((key >> (3 * k + d)) & 1) << k
        sh = np.array([sx, sy, sz])
        w = L / (1 << sh).astype(np.float64)
        cc = np.array(c) >> (tr.m - sh)                       # cell index at this level
        return np.array(lo) + cc * w, w

    off = 0
    for a in range(tr.nleaf):
        oa, wa = cell(a)
        la = tr.leaves[a][0]
        for b, code in nbr[a]:
            ob, wb = cell(b)
            lb, _, sb, cb = tr.leaves[b]
            S = np.array([code % 3 - 1, code // 3 % 3 - 1, code // 9 - 1], np.float64) * L
            seg = red[off:off + cb]
            off += cb
            # adjacency (closed): b + S overlaps D(a) or a - S overlaps D(b), positive volume
            def overlap(x0, w0, y0, wy):
                return np.all(np.minimum(x0 + w0, y0 + 2 * wy) - np.maximum(x0, y0 - wy) > 1e-12 * L)
            assert overlap(ob + S, wb, oa, wa) or overlap(oa - S, wa, ob, wb)
            for rec in seg:
                j = by_mass[float(rec[3])]
                back = rec[:3] + oa - S
                assert np.all(np.abs(back - inp.pos[j]) <= 1e-12 * (L + np.abs(oa)))
                assert np.all(inp.pos[j] >= ob - 1e-12 * L) and np.all(inp.pos[j] < ob + wb + 1e-12 * L)
                if lb >= la:
                    assert np.all(rec[:3] >= -wa * (1 + 1e-9)) and np.all(rec[:3] < 2 * wa * (1 + 1e-9))
    assert off == len(red)
