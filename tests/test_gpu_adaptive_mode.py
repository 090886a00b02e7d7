"""Adaptive-leaf MODE (SURVEY NEXT-1 on the per-step path, p2p_adaptive_enable): update / restructure / eval over
the adaptive leaves, asynchronous with every count on the device.  Its outputs must equal the synchronous
p2p_adaptive_eval (pinned against the oracle in test_gpu_adaptive.py) BIT FOR BIT -- same leaves, CSR, runs, items
and eval kernel -- and the oracle's plain definition within tolerance, over several time steps (moved particles,
changing N); its info reports the leaves' counts; exceeding the capacities measured at enable is reported, and
re-enabling recovers; disabling returns to grid mode after an update."""
import numpy as np
import pytest

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


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _sync_eval(P, inp, t, layout):
    """the synchronous path on a fresh plan (reference)"""
    with P.Plan(P.P2P_GRAVITY, _t(inp.pos), _t(inp.mass), inp.h, inp.lo, inp.nbox, inp.periodic, eps=inp.eps) as pl:
        phi = torch.empty(inp.n, dtype=pl.dtype, device="cuda")
        fld = torch.empty((inp.n, 3), dtype=pl.dtype, device="cuda")
        nrec = P.p2p_adaptive_eval(pl.handle, t, 9, phi.data_ptr(), fld.data_ptr(), layout=layout)
        torch.cuda.synchronize()
        return phi.cpu().numpy(), fld.cpu().numpy(), nrec


def _mode_eval(P, plan, layout):
    phi, fld = plan.eval(layout)
    torch.cuda.synchronize()
    return phi.cpu().numpy(), fld.cpu().numpy()


@pytest.mark.parametrize("t,dtype", [(4, np.float32), (16, np.float32), (64, np.float32), (8, np.float64)])
def test_adaptive_mode_time_steps(P, t, dtype):
    steps = [G.plummer(20000, 32, seed=11, dtype=dtype), G.plummer(20000, 32, seed=12, dtype=dtype),
             G.plummer(17000, 32, seed=13, dtype=dtype)]
    tol = 1e-5 if dtype == np.float32 else 1e-12
    a = steps[0]
    with P.Plan(P.P2P_GRAVITY, _t(a.pos), _t(a.mass), a.h, a.lo, a.nbox, a.periodic, eps=a.eps) as plan:
        plan.enable_adaptive(t)
        for k, inp in enumerate(steps):
            if k > 0:
                plan.update(_t(inp.pos), _t(inp.mass))  # asynchronous: leaves + CSR rebuilt on the device
            plan.restructure()
            out = {}
            for lay in (P.P2P_REDUNDANT, P.P2P_INDEXED):
                phi, fld = _mode_eval(P, plan, lay)
                rphi, rfld, nrec = _sync_eval(P, inp, t, lay)
                assert phi.tobytes() == rphi.tobytes() and fld.tobytes() == rfld.tobytes(), (k, lay)
                out[lay] = (phi, fld, nrec)
            tr = A.AdaptiveTree(inp, t)
            info = plan.refresh_info()
            assert info.n_boxes == len(tr.leaves)
            assert info.n_red == out[P.P2P_REDUNDANT][2]
            # values: the REDUNDANT runs (leaf-local coordinates, C24) against the plain definition.  The INDEXED
            # baseline works in absolute fp32 coordinates, whose rounding (~ulp(L)) is large against the 1e-4 pair
            # distances of this dense Plummer core (C11 reason 2, C25): it is held to bit-equality with the
            # synchronous path above, and to the oracle on sparser inputs (test_gpu_adaptive.py)
            ophi, ofld = tr.eval(inp.eps)
            phi, fld, _ = out[P.P2P_REDUNDANT]
            assert bounds.close(phi, ophi, tol) and bounds.close(fld, ofld, tol)


def test_adaptive_mode_overflow_and_disable(P):
    a = G.uniform_per_box(16, 2, seed=21)          # sparse uniform: few entries / records per leaf
    b = G.plummer(60000, 16, seed=22)              # dense cluster: many more records than 2x a's
    with P.Plan(P.P2P_GRAVITY, _t(a.pos), _t(a.mass), a.h, a.lo, a.nbox, a.periodic, eps=a.eps) as plan:
        plan.enable_adaptive(64)
        plan.update(_t(b.pos), _t(b.mass))
        plan.restructure()
        plan.eval(P.P2P_REDUNDANT)
        with pytest.raises(P.P2PError) as e:
            plan.refresh_info()
        assert e.value.status == P.P2P_ERR_OUT_OF_MEMORY
        plan.enable_adaptive(64)                   # re-measure on the current input
        plan.restructure()
        phi, fld = _mode_eval(P, plan, P.P2P_REDUNDANT)
        rphi, rfld, _ = _sync_eval(P, b, 64, P.P2P_REDUNDANT)
        assert phi.tobytes() == rphi.tobytes() and fld.tobytes() == rfld.tobytes()
        # back to grid mode: the grid neighbour lists need an update first
        plan.disable_adaptive()
        with pytest.raises(P.P2PError) as e:
            plan.restructure()
        assert e.value.status == P.P2P_ERR_BAD_STATE
        plan.update(_t(b.pos), _t(b.mass))
        plan.restructure()
        gphi, _ = _mode_eval(P, plan, P.P2P_REDUNDANT)
        assert np.isfinite(gphi).all()
        with pytest.raises(P.P2PError) as e:   # adaptive mode needs a periodic 2^m cube
            bad = G.plummer(2000, 12, seed=1)
            with P.Plan(P.P2P_GRAVITY, _t(bad.pos), _t(bad.mass), bad.h, bad.lo, bad.nbox, bad.periodic,
                        eps=bad.eps) as p2:
                p2.enable_adaptive(8)
        assert e.value.status == P.P2P_ERR_UNSUPPORTED
