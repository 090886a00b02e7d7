"""SURVEY NEXT-3 (VERDICT r1 missing #1): the per-thread dispersion D of P:L165 (§3.4) that scripts/locality_model.py
computes from the product's CSR, pinned against a brute force on the ORACLE's structures: mark every record a
target thread of box b reads (its neighbour segments) in a boolean array over the sorted particles and count the
maximal runs of marked records.  Also the closed forms of C1 (every box full, periodic 4^3)."""
import importlib.util
import os

import numpy as np
import pytest

import oracle
import p2p_inputs as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lm():
    spec = importlib.util.spec_from_file_location("locality_model", os.path.join(ROOT, "scripts", "locality_model.py"))
    mod = importlib.util.module_from_spec(spec)
    try:
        spec.loader.exec_module(mod)
    except SystemExit:
        pass
    return mod


def brute_D(gp):
    n = int(gp.bstart[-1])
    out = []
    for b in range(gp.B):
        mark = np.zeros(n + 2, bool)
        for e in range(gp.nbr_off[b], gp.nbr_off[b + 1]):
            k = gp.nbr_box[e]
            mark[1 + gp.bstart[k]:1 + gp.bstart[k + 1]] = True
        out.append(int(np.count_nonzero(mark[1:] & ~mark[:-1])))
    return np.array(out)


@pytest.mark.parametrize("inp", [G.uniform_per_box(4, 16, seed=0), G.random_gravity(2500, 0, seed=5, periodic=0b101,
                                                                                      nbox=(5, 7, 6), h=0.13),
                                 G.plummer(6000, 8, seed=2)], ids=["c1", "ragged", "plummer"])
def test_dispersion_per_thread_matches_brute_force(lm, inp):
    gp = oracle.GravityPlan(inp, with_red=False)
    D_box, thr = lm.dispersion_per_thread(gp.nbr_off, gp.nbr_box, gp.bstart)
    assert np.array_equal(D_box, brute_D(gp))
    assert np.array_equal(thr, np.diff(gp.bstart.astype(np.int64)))
    assert np.all(D_box >= 1) and np.all(D_box <= np.diff(gp.nbr_off.astype(np.int64)))


def test_dispersion_closed_forms(lm):
    """one box: D = 1; a line of 8 occupied boxes along x (open), Morton order = x order, so every box's 3 (ends: 2)
    neighbours are consecutive records: D = 1; the same line with every other box empty: the neighbours of an
    occupied box are itself only (D = 1); a periodic 4-line: the end boxes read boxes {3, 0, 1} = two blocks"""
    rng = np.random.default_rng(0)

    def line(nx, occupied, per):
        pts = []
        for x in occupied:
            p = np.column_stack([x + rng.uniform(0.1, 0.9, 5), rng.uniform(0.1, 0.9, 5), rng.uniform(0.1, 0.9, 5)]) / nx
            pts.append(p)
        pos = np.concatenate(pts)
        return G.GravityInput(pos, np.ones(len(pos)) / len(pos), (0.0, 0.0, 0.0), 1.0 / nx, (nx, 1, 1), per, 1e-3)

    for inp, want in [(line(1, [0], 0), [1]), (line(8, range(8), 0), [1] * 8), (line(8, [0, 2, 4, 6], 0), [1] * 4),
                      (line(4, range(4), 0b001), [2, 1, 1, 2])]:
        gp = oracle.GravityPlan(inp, with_red=False)
        D_box, thr = lm.dispersion_per_thread(gp.nbr_off, gp.nbr_box, gp.bstart)
        assert D_box.tolist() == want and np.all(thr == 5)
        assert np.array_equal(D_box, brute_D(gp))
