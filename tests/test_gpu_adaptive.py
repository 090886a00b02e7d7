"""SURVEY NEXT-1 on the GPU (-m gpu): the adaptive binary-tree leaves (DESIGN C22, p2p_adaptive_leaves) and their
closed neighbour CSR (C23, p2p_adaptive_neighbours) equal the pinned oracle's (oracle/adaptive.py) bit for bit --
prefix length, prefix and first sorted particle of every leaf in Morton order; every leaf's (neighbour leaf, image
code) list in order -- on clustered and uniform inputs, for several clustering thresholds, after p2p_plan_update
too; plans that are not a periodic 2^m cube are rejected."""
import numpy as np
import pytest

import oracle
import p2p_bounds as bounds
import p2p_inputs as G
from oracle import adaptive as A

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2511_21535_b200 as P
    return P


def _plan(P, inp):
    pos = torch.from_numpy(inp.pos).cuda()
    m = torch.from_numpy(inp.mass).cuda()
    return P.Plan(P.P2P_GRAVITY, pos, m, inp.h, inp.lo, inp.nbox, inp.periodic, eps=inp.eps)


def _check(P, plan, inp, t, min_bits=9):
    ln, px, st = P.p2p_adaptive_leaves(plan.handle, t, min_bits, plan.info.n_boxes)
    tr = A.AdaptiveTree(inp, t, min_bits)
    want = np.array([(l, p, s) for l, p, s, _ in tr.leaves], dtype=np.int64).reshape(-1, 3)
    got = np.stack([ln, px, st], axis=1).astype(np.int64)
    assert got.shape == want.shape and np.array_equal(got, want)


@pytest.mark.parametrize("t", [1, 4, 16, 64, 1000])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_plummer(P, t, dtype):
    inp = G.plummer(20000, 32, seed=2, dtype=dtype)
    with _plan(P, inp) as plan:
        _check(P, plan, inp, t)


def test_uniform_and_min_bits(P):
    inp = G.uniform_per_box(16, 3, seed=4)
    with _plan(P, inp) as plan:
        _check(P, plan, inp, 3)              # every finest box its own leaf
        _check(P, plan, inp, 24, 0)          # 8 boxes per leaf from the root down
        _check(P, plan, inp, 10**6, 0)       # the root alone


def test_after_update_and_large(P):
    a = G.plummer(5000, 64, seed=5)
    b = G.plummer(300000, 64, seed=6)
    with _plan(P, a) as plan:
        plan.update(torch.from_numpy(b.pos).cuda(), torch.from_numpy(b.mass).cuda())
        plan.refresh_info()
        _check(P, plan, b, 8)


def test_rejects_non_cube(P):
    inp = G.random_gravity(2000, 0, seed=1, periodic=0b111, nbox=(8, 8, 6), h=0.125)
    with _plan(P, inp) as plan:
        with pytest.raises(P.P2PError):
            P.p2p_adaptive_leaves(plan.handle, 4, 9, plan.info.n_boxes)


def _check_csr(P, plan, inp, t, min_bits=9):
    B = plan.info.n_boxes
    off, nbr, code = P.p2p_adaptive_neighbours(plan.handle, t, min_bits, B + 1, 27 * 64 * B)
    tr = A.AdaptiveTree(inp, t, min_bits)
    want = tr.neighbours()
    assert len(off) == tr.nleaf + 1 and off[0] == 0
    for a in range(tr.nleaf):
        got = list(zip(nbr[off[a]:off[a + 1]].tolist(), code[off[a]:off[a + 1]].tolist()))
        assert got == want[a], a


@pytest.mark.parametrize("seed,t", [(1, 8), (2, 16), (4, 3), (5, 64)])
def test_neighbour_csr_plummer(P, seed, t):
    inp = G.plummer(3000, 32, seed=seed)
    with _plan(P, inp) as plan:
        _check_csr(P, plan, inp, t)


def test_neighbour_csr_uniform_is_the_stencil(P):
    inp = G.uniform_per_box(8, 4, seed=5)
    with _plan(P, inp) as plan:
        off, nbr, code = P.p2p_adaptive_neighbours(plan.handle, 4, 9, 513, 27 * 512)
        assert np.all(np.diff(off) == 27)
        _check_csr(P, plan, inp, 4)


@pytest.mark.parametrize("seed,t,dtype", [(1, 8, np.float32), (2, 16, np.float32), (3, 3, np.float32),
                                          (4, 32, np.float64)])
def test_adaptive_red_and_eval(P, seed, t, dtype):
    """C24 runs bit-exact vs the oracle; potentials / fields vs the oracle's plain definition (1e-5 / 1e-12)"""
    inp = G.plummer(3000, 32, seed=seed, dtype=dtype)
    tr = A.AdaptiveTree(inp, t)
    want_red = tr.red(dtype)
    with _plan(P, inp) as plan:
        red = np.empty((want_red.shape[0] + 1, 4), dtype)
        n = P.p2p_adaptive_eval(plan.handle, t, 9, None, None, red)
        assert n == want_red.shape[0]
        assert red[:n].tobytes() == want_red.tobytes()
        phi = torch.empty(inp.n, dtype=torch.from_numpy(np.zeros(1, dtype)).dtype, device="cuda")
        fld = torch.empty((inp.n, 3), dtype=phi.dtype, device="cuda")
        P.p2p_adaptive_eval(plan.handle, t, 9, phi.data_ptr(), fld.data_ptr())
        torch.cuda.synchronize()
        phi, fld = phi.cpu().numpy(), fld.cpu().numpy()
    rphi, rf = tr.eval(inp.eps)
    tol = 1e-5 if dtype == np.float32 else 1e-12
    assert bounds.close(phi, rphi, tol) and bounds.close(fld, rf, tol)


def test_adaptive_equal_leaves_match_the_grid_path(P):
    """equal leaves: the adaptive path's outputs are the grid REDUNDANT path's, up to summation order"""
    inp = G.uniform_per_box(16, 4, seed=8)
    with _plan(P, inp) as plan:
        plan.restructure()
        gphi, gf = [x.cpu().numpy() for x in plan.eval(P.P2P_REDUNDANT)]
        phi = torch.empty(inp.n, device="cuda")
        fld = torch.empty((inp.n, 3), device="cuda")
        P.p2p_adaptive_eval(plan.handle, 4, 9, phi.data_ptr(), fld.data_ptr())
        torch.cuda.synchronize()
    assert bounds.close(phi.cpu().numpy(), gphi, 1e-6) and bounds.close(fld.cpu().numpy(), gf, 1e-6)


def test_full_size_sampled(P):
    """BASELINE configs[2] (10^6 Plummer, 128^3 finest boxes), t = 16: the CSR rows and the potentials / fields of
    120 seeded-random leaves (and the 10 largest) against the oracle's per-leaf definition"""
    inp = G.config("c3")
    t = 16
    tr = A.AdaptiveTree(inp, t)
    with _plan(P, inp) as plan:
        B = plan.info.n_boxes
        off, nbr, code = P.p2p_adaptive_neighbours(plan.handle, t, 9, B + 1, 40 * B)
        phi = torch.empty(inp.n, device="cuda")
        fld = torch.empty((inp.n, 3), device="cuda")
        P.p2p_adaptive_eval(plan.handle, t, 9, phi.data_ptr(), fld.data_ptr())
        torch.cuda.synchronize()
        phi, fld = phi.cpu().numpy(), fld.cpu().numpy()
    assert len(off) == tr.nleaf + 1
    rng = np.random.default_rng(0)
    cnt = np.array([c for _, _, _, c in tr.leaves])
    pick = np.unique(np.concatenate([rng.choice(tr.nleaf, 120, replace=False), np.argsort(cnt)[-10:]]))
    e = np.zeros(4)   # squared error / norm of phi, then of the field (one 3n vector)
    for a in pick:
        want = A.neighbours_of(tr, int(a))
        assert list(zip(nbr[off[a]:off[a + 1]].tolist(), code[off[a]:off[a + 1]].tolist())) == want
        ti, p, f = A.eval_leaf(tr, int(a), inp.eps, want)
        e += [((phi[ti] - p) ** 2).sum(), (p ** 2).sum(), ((fld[ti] - f) ** 2).sum(), (f ** 2).sum()]
    assert np.sqrt(e[0] / e[1]) <= 1e-5 and np.sqrt(e[2] / e[3]) <= 1e-5


def test_adaptive_errors_and_determinism(P):
    inp = G.plummer(4000, 32, seed=11)
    with _plan(P, inp) as plan:
        B = plan.info.n_boxes
        with pytest.raises(P.P2PError):           # min_bits < 9: periodic images not unique
            P.p2p_adaptive_neighbours(plan.handle, 8, 6, B + 1, 64 * B)
        with pytest.raises(P.P2PError):           # t < 1
            P.p2p_adaptive_leaves(plan.handle, 0, 9, B)
        with pytest.raises(P.P2PError):           # entry capacity too small
            P.p2p_adaptive_neighbours(plan.handle, 8, 9, B + 1, 10)
        runs = []
        for _ in range(3):                       # the transposed entries are sorted: CSR and outputs are bitwise stable
            off, nbr, code = P.p2p_adaptive_neighbours(plan.handle, 8, 9, B + 1, 64 * B)
            phi = torch.empty(inp.n, device="cuda")
            fld = torch.empty((inp.n, 3), device="cuda")
            P.p2p_adaptive_eval(plan.handle, 8, 9, phi.data_ptr(), fld.data_ptr())
            torch.cuda.synchronize()
            runs.append((off.tobytes(), nbr.tobytes(), code.tobytes(), phi.cpu().numpy().tobytes(),
                         fld.cpu().numpy().tobytes()))
        assert runs[0] == runs[1] == runs[2]
        # the plan itself is untouched: the grid path still evaluates as before
        plan.restructure()
        gphi, _ = plan.eval(P.P2P_REDUNDANT)
        assert torch.isfinite(gphi).all()


@pytest.mark.parametrize("seed,t,dtype", [(1, 8, np.float32), (3, 3, np.float32), (4, 32, np.float64),
                                          (6, 64, np.float32)])
def test_adaptive_indexed_baseline(P, seed, t, dtype):
    """the non-redundant baseline on the leaves (rows longer than a warp included) vs the oracle and vs REDUNDANT"""
    inp = G.plummer(3000, 32, seed=seed, dtype=dtype)
    tr = A.AdaptiveTree(inp, t)
    assert max(len(x) for x in tr.neighbours()) > 32
    tdt = torch.float32 if dtype == np.float32 else torch.float64
    out = {}
    with _plan(P, inp) as plan:
        for lay in (P.P2P_REDUNDANT, P.P2P_INDEXED):
            phi = torch.empty(inp.n, dtype=tdt, device="cuda")
            fld = torch.empty((inp.n, 3), dtype=tdt, device="cuda")
            P.p2p_adaptive_eval(plan.handle, t, 9, phi.data_ptr(), fld.data_ptr(), layout=lay)
            torch.cuda.synchronize()
            out[lay] = (phi.cpu().numpy(), fld.cpu().numpy())
    rphi, rf = tr.eval(inp.eps)
    tol = 1e-5 if dtype == np.float32 else 1e-12
    for lay, (phi, fld) in out.items():
        assert bounds.close(phi, rphi, tol) and bounds.close(fld, rf, tol), lay


def _shifted(inp, lo):
    """the same clustered particles in a domain at origin lo (positions moved in fp64, rounded once)"""
    import dataclasses
    pos = (inp.pos.astype(np.float64) + np.asarray(lo)).astype(inp.pos.dtype)
    return dataclasses.replace(inp, pos=np.ascontiguousarray(pos), lo=tuple(lo), name=inp.name + f" lo={lo}")


@pytest.mark.parametrize("lo,t,maxgrid", [((0.1, -0.37, 0.55), 8, None),     # leaf origins not fp32 values: fp64
                                          ((0.25, 0.5, -0.75), 16, None),    # fp32-exact origins: fp32 fast path
                                          ((0.0, 0.0, 0.0), 4, "2"),         # 16 warps walk every chunk
                                          ((0.1, -0.37, 0.55), 32, "3")])
def test_adaptive_runs_origin_and_chunk_walk(P, lo, t, maxgrid, monkeypatch):
    """C24 runs bit-exact vs the oracle with the domain off the origin -- both rounding paths of the chunk
    restructure (the fp64 sequence, and the fp32 subtraction taken when every lattice origin is an fp32 value) --
    and with the grid capped so that each warp walks many chunks (its one-chunk-ahead loads)"""
    if maxgrid:
        monkeypatch.setenv("P2P_RS_MAXGRID", maxgrid)
    inp = _shifted(G.plummer(6000, 32, seed=31), lo)
    tr = A.AdaptiveTree(inp, t)
    want_red = tr.red(np.float32)
    with _plan(P, inp) as plan:
        red = np.empty((want_red.shape[0] + 1, 4), np.float32)
        n = P.p2p_adaptive_eval(plan.handle, t, 9, None, None, red)
        assert n == want_red.shape[0]
        assert red[:n].tobytes() == want_red.tobytes()
        # the asynchronous mode builds the same runs (its eval equals the synchronous one bit for bit)
        plan.enable_adaptive(t)
        phi, fld = [x.cpu().numpy() for x in plan.eval(P.P2P_INDEXED)]  # INDEXED needs the update only
        with pytest.raises(P.P2PError) as e:
            plan.eval(P.P2P_REDUNDANT)
        assert e.value.status == P.P2P_ERR_BAD_STATE
        info = plan.refresh_info()  # counts are the update's: known before the restructure
        assert info.n_red == n
        plan.restructure()
        mphi, mfld = [x.cpu().numpy() for x in plan.eval(P.P2P_REDUNDANT)]
    sphi = torch.empty(inp.n, device="cuda")
    sfld = torch.empty((inp.n, 3), device="cuda")
    with _plan(P, inp) as plan:
        P.p2p_adaptive_eval(plan.handle, t, 9, sphi.data_ptr(), sfld.data_ptr())
        torch.cuda.synchronize()
    assert mphi.tobytes() == sphi.cpu().numpy().tobytes() and mfld.tobytes() == sfld.cpu().numpy().tobytes()
    rphi, rf = tr.eval(inp.eps)
    assert bounds.close(mphi, rphi, 1e-5) and bounds.close(mfld, rf, 1e-5)
    assert np.isfinite(phi).all()


@pytest.mark.parametrize("t,cap", [(2, "1"), (4, "1"), (8, "1"), (4, "0")])
def test_adaptive_quads(P, t, cap, monkeypatch):
    """multi-leaf quad items (REDUNDANT, fp32; opt-in P2P_ADAPT_QUADS=1): within tolerance of the oracle with and
    without them, and actually taken (the 8-lane split of a quad leaf sums in another order than its own item)"""
    monkeypatch.setenv("P2P_ADAPT_CAP", cap)  # "0": uncapped REDUNDANT items, quads limited by 8 targets / 16 bits
    inp = G.plummer(8000, 32, seed=40 + t)
    tr = A.AdaptiveTree(inp, t)
    rphi, rf = tr.eval(inp.eps)
    out = []
    for quads in ("1", "0"):
        monkeypatch.setenv("P2P_ADAPT_QUADS", quads)
        phi = torch.empty(inp.n, device="cuda")
        fld = torch.empty((inp.n, 3), device="cuda")
        with _plan(P, inp) as plan:
            P.p2p_adaptive_eval(plan.handle, t, 9, phi.data_ptr(), fld.data_ptr())
            torch.cuda.synchronize()
        phi, fld = phi.cpu().numpy(), fld.cpu().numpy()
        assert bounds.close(phi, rphi, 1e-5) and bounds.close(fld, rf, 1e-5)
        out.append(phi.tobytes() + fld.tobytes())
    assert out[0] != out[1]
