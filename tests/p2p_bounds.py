"""Error bounds of the GPU-vs-oracle parity tests (tests only).

north_star's bar is the whole-array relative L2 error (<= 1e-5 fp32, <= 1e-12 fp64).  Beside it every
comparison also bounds the error PER ELEMENT, so an error confined to one box of a large sample cannot hide in
the norm: for every particle i (a row: phi_i, the field vector a_i, the complex y_i)

    |g_i - o_i| / max(|o_i|, FLOOR * rms_j |o_j|)  <=  ELEM_FACTOR * tol

The floor only matters where the reference itself nearly vanishes by cancellation (a field component sum of
opposite terms, an isolated particle's phi = 0); there the bound is relative to the array's scale.  Complex
Helmholtz outputs y_i = sum_j P_ij x_j with x ~ CN(0,1) (C17) are random-phase sums: |y_i| is Rayleigh-distributed,
so a fixed fraction of the elements nearly cancels (P(|y| < 0.01 rms) ~ 1e-4: hundreds of elements at c2b), while a
sum's rounding error scales with the sum of |terms| ~ rms, not with |y_i|.  Their floor is therefore the rms
itself (COMPLEX_FLOOR): the per-element check bounds max_i |g_i - o_i| / max(|o_i|, rms).  With
P2P_BOUNDS_LOG=<file> every check appends its two measured errors (calibration record, see profiles/)."""
import json
import os

import numpy as np

ELEM_FACTOR = 10.0
FLOOR = 1e-2
COMPLEX_FLOOR = 1.0


def _rows(a):
    a = np.asarray(a)
    if np.iscomplexobj(a):
        return np.abs(a.astype(np.complex128))
    a = a.astype(np.float64)
    if a.ndim == 1:
        return np.abs(a)
    return np.sqrt((a.reshape(a.shape[0], -1) ** 2).sum(axis=1))


def errors(g, o):
    g = np.asarray(g)
    o = np.asarray(o)
    if np.iscomplexobj(o) and not np.iscomplexobj(g):
        g = g[..., 0] + 1j * g[..., 1] if g.ndim >= 2 and g.shape[-1] == 2 else g
    g = g.astype(o.dtype if np.iscomplexobj(o) else np.float64).reshape(o.shape)
    d = g - o
    den = np.sqrt((np.abs(o.astype(np.complex128) if np.iscomplexobj(o) else o.astype(np.float64)) ** 2).sum())
    l2 = float(np.sqrt((np.abs(d) ** 2).sum()) / den) if den > 0 else float(np.sqrt((np.abs(d) ** 2).sum()))
    ro = _rows(o)
    if ro.size == 0:
        return l2, 0.0
    rms = float(np.sqrt((ro ** 2).mean()))
    scale = np.maximum(ro, (COMPLEX_FLOOR if np.iscomplexobj(o) else FLOOR) * rms)
    rd = _rows(d)
    elem = float((rd / np.where(scale > 0, scale, 1.0)).max())
    return l2, elem


def close(g, o, tol, what=""):
    """True iff the relative L2 error <= tol AND the per-element error <= ELEM_FACTOR * tol"""
    l2, elem = errors(g, o)
    log = os.environ.get("P2P_BOUNDS_LOG")
    if log:
        with open(log, "a") as f:
            f.write(json.dumps({"test": os.environ.get("PYTEST_CURRENT_TEST", "").split(" ")[0], "what": what,
                                "tol": tol, "rel_l2": l2, "elem": elem, "n": int(np.asarray(o).shape[0])}) + "\n")
    ok = l2 <= tol and elem <= ELEM_FACTOR * tol
    if not ok:
        print(f"bounds failed {what}: rel_l2 {l2:.3e} (tol {tol:.1e}), per-element {elem:.3e} "
              f"(bound {ELEM_FACTOR * tol:.1e})")
    return ok
