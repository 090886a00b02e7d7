"""Pins of the Helmholtz (DBIM-like) oracle against scipy's Hankel functions, numerical quadrature of the
self-cell integral, the SURVEY §8c worked example, closed-form neighbour counts, table reciprocity and the
list-free dense masked matvec.  CPU only."""
import json
import math
import os

import numpy as np
import pytest

import oracle
import p2p_inputs as G

GOLD = os.path.join(os.path.dirname(__file__), "golden")
sp = pytest.importorskip("scipy.special")


def test_weight_matches_scipy_hankel():
    # G(r) Delta^2 = (i/4) H0^(1)(k r) Delta^2 (C15), glibc y0/j0 vs scipy hankel1
    delta, k = 0.7, 2 * math.pi / 7.0
    for r in [0.3, 1.0, 1.2345, math.sqrt(2) * 0.7, 5.0, 17.0]:
        ref = 0.25j * sp.hankel1(0, k * r) * delta * delta
        got = oracle.helm_weight(r, delta, k)
        assert abs(got - ref) <= 1e-14 * abs(ref)


def test_self_term_closed_form_and_quadrature():
    from scipy import integrate
    delta = 1.0
    k = 2 * math.pi / 10
    a = delta / math.sqrt(math.pi)
    got = oracle.helm_weight(0.0, delta, k)
    closed = (1j * math.pi * a / (2 * k)) * sp.hankel1(1, k * a) - 1 / k ** 2
    # integral of (i/4) H0^(1)(k rho) over the equal-area disk, by quadrature (log singularity at 0)
    re = integrate.quad(lambda r: (-0.25 * sp.y0(k * r)) * 2 * math.pi * r, 0, a, limit=200, epsabs=1e-15)[0]
    im = integrate.quad(lambda r: (0.25 * sp.j0(k * r)) * 2 * math.pi * r, 0, a, limit=200, epsabs=1e-15)[0]
    gold = json.load(open(os.path.join(GOLD, "helmholtz_worked_example.json")))
    assert abs(got - closed) < 1e-15
    assert abs(got - complex(re, im)) < 1e-12
    assert abs(got - complex(*gold["self"])) < 1e-15


def test_worked_example_t1_3x3():
    gold = json.load(open(os.path.join(GOLD, "helmholtz_worked_example.json")))
    pos = np.array([[x + 0.5, y + 0.5] for y in range(3) for x in range(3)], np.float32)
    inp = G.HelmholtzInput(pos, np.ones(9, np.complex64), (0.0, 0.0), 1.0, (3, 3), 1, 1.0, 2 * math.pi / 10)
    hp = oracle.HelmholtzPlan(inp)
    for y in (hp.eval_table(), oracle.helm_dense(inp)):
        assert abs(y[4] - complex(*gold["y_centre"])) < 1e-14
        for e in (1, 3, 5, 7):
            assert abs(y[e] - complex(*gold["y_edge"])) < 1e-14
        for c in (0, 2, 6, 8):
            assert abs(y[c] - complex(*gold["y_corner"])) < 1e-14
    assert abs(hp.P[0, 4 * 1 + 0] - complex(*gold["self"])) < 1e-15
    assert abs(hp.P[0, 5] - complex(*gold["G1_delta2"])) < 1e-15
    assert abs(hp.P[0, 8] - complex(*gold["Gsqrt2_delta2"])) < 1e-15


def test_table_reciprocity():
    # P[i][s, j] = P[j][s_bar, i], s_bar the opposite stencil slot (8 - s)
    for t in (4, 16):
        P = oracle.helm_table(t, 1.0, 2 * math.pi / 10).reshape(t, 9, t)
        assert np.allclose(P, np.transpose(P[:, ::-1, :], (2, 1, 0)), rtol=0, atol=1e-15)


def test_neighbour_counts_closed_form():
    # open n x n grid: sum_b |N(b)| = 9(n-2)^2 + 24(n-2) + 16; interior 9, edge 6, corner 4
    for n in (3, 8):
        hp = oracle.HelmholtzPlan(G.dbim_lattice(n, 4, seed=0))
        cnt = np.count_nonzero(hp.nbr9 != 0xFFFFFFFF, axis=1)
        assert cnt.sum() == 9 * (n - 2) ** 2 + 24 * (n - 2) + 16
        assert sorted(set(cnt.tolist())) == sorted({4, 6, 9} if n > 2 else {4})
    assert 9 * 254 ** 2 + 24 * 254 + 16 == 586756      # C2 (256^2 boxes) count quoted in SURVEY §8a


def test_subcell_key_order():
    # in-box order equals the pattern-table index j = sy*st + sx (C8)
    inp = G.dbim_lattice(4, 16, seed=1)
    hp = oracle.HelmholtzPlan(inp)
    st = 4
    for b in range(hp.B):
        p = inp.pos[hp.perm[hp.bstart[b]:hp.bstart[b + 1]]].astype(np.float64)
        o = np.floor(p[0] / (st * inp.delta)) * st * inp.delta
        q = np.floor((p - o) / inp.delta).astype(int)
        assert np.array_equal(q[:, 1] * st + q[:, 0], np.arange(16))


@pytest.mark.parametrize("t,holes", [(16, None), (4, [(1, 1), (3, 0)]), (1, None)])
def test_table_eval_matches_dense(t, holes):
    inp = G.dbim_lattice(4, t, seed=2, holes=holes)
    hp = oracle.HelmholtzPlan(inp)
    y = hp.eval_table()
    yd = oracle.helm_dense(inp)
    assert oracle.rel_l2(y, yd) < 1e-13
    # Xg path: y_b = P @ Xg[b].ravel()
    Xg = hp.xg()
    yb = np.einsum("im,bm->bi", hp.P, Xg.reshape(hp.B, -1))
    ys = np.zeros_like(y)
    ys[hp.perm] = yb.ravel()
    assert oracle.rel_l2(ys, yd) < 1e-13


def test_bilinear_reciprocity():
    # the near-field operator is complex symmetric: u^T (A v) = v^T (A u)
    base = G.dbim_lattice(4, 16, seed=5)
    rng = np.random.default_rng(0)
    u = (rng.normal(size=base.n) + 1j * rng.normal(size=base.n)).astype(np.complex64)
    v = (rng.normal(size=base.n) + 1j * rng.normal(size=base.n)).astype(np.complex64)
    Av = oracle.helm_dense(G.HelmholtzInput(base.pos, v, base.lo, base.h, base.nbox, base.t, base.delta, base.k))
    Au = oracle.helm_dense(G.HelmholtzInput(base.pos, u, base.lo, base.h, base.nbox, base.t, base.delta, base.k))
    lhs, rhs = np.dot(u.astype(np.complex128), Av), np.dot(v.astype(np.complex128), Au)
    assert abs(lhs - rhs) <= 1e-13 * abs(lhs)


def test_irregular_lattice_rejected():
    inp = G.dbim_lattice(3, 4, seed=0)
    pos = inp.pos.copy()
    pos[0] = pos[1]                                   # two samples in one sub-cell
    bad = G.HelmholtzInput(pos, inp.x, inp.lo, inp.h, inp.nbox, inp.t, inp.delta, inp.k)
    with pytest.raises(oracle.Unsupported):
        oracle.HelmholtzPlan(bad)
