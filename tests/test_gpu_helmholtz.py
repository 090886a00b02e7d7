"""GPU parity of the Helmholtz (DBIM-like) path (-m gpu): structures bit-exact, y within 1e-5 (complex64) /
1e-12 (complex128) of the oracle.  REDUNDANT (im2col Xg) == INDEXED bit for bit on either execution unit: the
CUDA-core kernels, and for fp32 t in {16, 64} the 3xTF32 tensor-core GEMM (k_helm_tc.cu: REDUNDANT streams Xg by
TMA, INDEXED gathers the neighbour segments of the sorted unknowns by cp.async -- same A operand, same MMAs), which
is also held to its own error budget (<= 5e-6 relative L2)."""
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


def gpu_plan(P, inp, f64=False):
    rdt = torch.float64 if f64 else torch.float32
    pos = torch.from_numpy(inp.pos.astype(np.float64 if f64 else np.float32)).cuda()
    x = np.ascontiguousarray(inp.x.astype(np.complex128 if f64 else np.complex64))
    xr = torch.from_numpy(x.view(np.float64 if f64 else np.float32).reshape(-1, 2)).cuda().to(rdt)
    return P.Plan(P.P2P_HELMHOLTZ2D, pos, xr, inp.h, inp.lo, inp.nbox, 0, k=inp.k, t=inp.t)


def to_c(y):
    a = y.cpu().numpy()
    return a[:, 0] + 1j * a[:, 1]


@pytest.mark.parametrize("t,n,holes,f64", [(16, 8, None, False), (64, 6, None, False), (4, 5, [(1, 2)], False),
                                           (1, 7, None, False), (16, 6, [(0, 0), (3, 3)], True), (9, 4, None, True)])
def test_helmholtz_parity(P, t, n, holes, f64):
    inp = G.dbim_lattice(n, t, seed=t + n, holes=holes)
    hp = oracle.HelmholtzPlan(inp)
    ref = hp.eval_table()
    assert bounds.close(ref, oracle.helm_dense(inp), 1e-13)
    with gpu_plan(P, inp, f64) as plan:
        assert plan.info.n_boxes == hp.B
        assert plan.info.n_pairs == hp.n_pairs
        assert np.array_equal(plan.copy_out(P.P2P_ARR_PERM), hp.perm)
        assert np.array_equal(plan.copy_out(P.P2P_ARR_SORTED_KEYS), hp.skey)
        assert np.array_equal(plan.copy_out(P.P2P_ARR_BOX_KEYS), hp.bkey)
        assert np.array_equal(plan.copy_out(P.P2P_ARR_BOX_START), hp.bstart)
        assert np.array_equal(plan.copy_out(P.P2P_ARR_NBR_BOX), hp.nbr9.ravel())
        plan.restructure()
        Xg = plan.copy_out(P.P2P_ARR_RED).reshape(hp.B, 9, t)
        assert np.array_equal(Xg, hp.xg().astype(Xg.dtype))   # zero-padded im2col, bit copies
        y_red = to_c(plan.eval(P.P2P_REDUNDANT))
        y_idx = to_c(plan.eval(P.P2P_INDEXED))
    tol = 1e-12 if f64 else 1e-5
    assert bounds.close(y_red, ref, tol)
    assert bounds.close(y_idx, ref, tol)
    if tensor_core_path(t, f64):
        assert bounds.close(y_red, ref, 5e-6)
    assert np.array_equal(y_red, y_idx)


def tensor_core_path(t, f64):
    return (not f64) and t in (16, 64)


@pytest.mark.parametrize("t,n,holes", [(16, 37, None), (64, 23, [(5, 7)]), (16, 12, [(0, 11), (11, 0)])])
def test_helmholtz_tensor_core_ragged(P, t, n, holes):
    """the tcgen05 GEMM on box counts that are not multiples of its 128-box tile (TMA zero-fill of the last
    tile's rows, masked epilogue) and with missing neighbours (zero segments of Xg)"""
    inp = G.dbim_lattice(n, t, seed=7 * n + t, holes=holes)
    hp = oracle.HelmholtzPlan(inp)
    ref = hp.eval_table()
    with gpu_plan(P, inp) as plan:
        plan.restructure()
        y_red = to_c(plan.eval(P.P2P_REDUNDANT))
        y_idx = to_c(plan.eval(P.P2P_INDEXED))
    assert bounds.close(y_red, ref, 5e-6)
    assert bounds.close(y_idx, ref, 1e-5)
    assert np.array_equal(y_red, y_idx)  # the tensor-core gather (INDEXED) feeds the GEMM the same A values
    # every output written (no stale values from a skipped tile row)
    assert np.isfinite(y_red).all() and np.abs(y_red).min() > 0


def test_irregular_rejected(P):
    inp = G.dbim_lattice(3, 4, seed=0)
    pos = inp.pos.copy()
    pos[0] = pos[1]
    bad = G.HelmholtzInput(pos, inp.x, inp.lo, inp.h, inp.nbox, inp.t, inp.delta, inp.k)
    with pytest.raises(P.P2PError) as e:
        gpu_plan(P, bad)
    assert e.value.status == P.P2P_ERR_UNSUPPORTED


def test_set_charges_dbim_iterations(P):
    """DBIM reuses the geometry across iterations: new unknowns, same plan"""
    inp = G.dbim_lattice(8, 16, seed=1)
    rng = np.random.default_rng(5)
    with gpu_plan(P, inp) as plan:
        for it in range(3):
            x = ((rng.normal(size=inp.n) + 1j * rng.normal(size=inp.n)) / np.sqrt(2)).astype(np.complex64)
            plan.set_charges(torch.from_numpy(x.view(np.float32).reshape(-1, 2)).cuda())
            plan.restructure()
            y = to_c(plan.eval(P.P2P_REDUNDANT))
            ref = oracle.HelmholtzPlan(G.HelmholtzInput(inp.pos, x, inp.lo, inp.h, inp.nbox, inp.t, inp.delta,
                                                        inp.k)).eval_table()
            assert bounds.close(y, ref, 1e-5)


def test_rf_copies_bitwise_equal(P, monkeypatch):
    """NEXT-2 block-level redundancy: RF copies of the tensor-core operand W give the RF = 1 result bit for
    bit (every CTA reads an identical copy)"""
    import numpy as np
    import p2p_inputs as G
    h = G.dbim_lattice(32, 64, seed=3)
    xr = torch.from_numpy(h.x.view(np.float32).reshape(-1, 2)).cuda()
    pos = torch.from_numpy(h.pos).cuda()
    out = []
    for rf in ("1", "2", "4"):
        monkeypatch.setenv("P2P_HELM_RF", rf)
        with P.Plan(P.P2P_HELMHOLTZ2D, pos, xr, h.h, h.lo, h.nbox, 0, k=h.k, t=h.t) as plan:
            plan.restructure()
            out.append(plan.eval(P.P2P_REDUNDANT).cpu().numpy().tobytes())
    assert out[0] == out[1] == out[2]


@pytest.mark.parametrize("t", [16, 64])
def test_tc_multicast_and_split(P, monkeypatch, t):
    """NEXT-2 on B200 clusters: the W operand multicast over clusters of 2 / 4 CTAs (TMA .multicast::cluster, multicast
    tcgen05.commit) stages the same operands and issues the same MMA sequence, so it gives the default's bits; the
    t = 64 output split over two CTAs accumulates its K slices over 6 instead of 3 TMEM accumulators (other rounding):
    REDUNDANT == INDEXED bitwise within it and the oracle bound.  A ragged box count (not a multiple of the 128-box
    tile, nor of the cluster) exercises the padding CTAs of the last cluster"""
    h = G.dbim_lattice(21, t, seed=5)  # 441 boxes: 3.4 tiles
    xr = torch.from_numpy(h.x.view(np.float32).reshape(-1, 2)).cuda()
    pos = torch.from_numpy(h.pos).cuda()
    out = {}
    with P.Plan(P.P2P_HELMHOLTZ2D, pos, xr, h.h, h.lo, h.nbox, 0, k=h.k, t=h.t) as plan:
        plan.restructure()
        for cl, ns in [("1", "1"), ("2", "1"), ("4", "1")] + ([("1", "2"), ("2", "2")] if t == 64 else []):
            monkeypatch.setenv("P2P_HELM_CLUSTER", cl)
            monkeypatch.setenv("P2P_HELM_NSPLIT", ns)
            for lay in ("redundant", "indexed"):
                out[(cl, ns, lay)] = plan.eval(P.LAYOUTS[lay]).cpu().numpy()
    for (cl, ns, lay), v in out.items():  # bitwise within each output split, for every cluster size and layout
        assert v.tobytes() == out[("1", ns, "redundant")].tobytes(), (cl, ns, lay)
    if t == 64:
        ref = oracle.HelmholtzPlan(h).eval_table()
        y = out[("1", "2", "redundant")]
        assert bounds.close(y[:, 0] + 1j * y[:, 1], ref, 5e-6)
