"""fp64 CPU oracle of the MLFMA near-field (P2P) operator -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` legs may import
this package.  The product path (paper_2511_21535_b200) never imports it, and this package never
imports the product: the only module both sides use is the seeded input generator p2p_inputs.

Python layer = argument marshalling over oracle/p2p_oracle.c (all arithmetic is in the C file, every
function there cites the PAPER.md / SPEC.md passage or DESIGN.md reading it follows).

Parity status: every function is pinned by tests/test_oracle_*.py against closed forms, brute force,
Newton's third law, library Bessel functions or the SURVEY §8c worked examples -- none is "parity
unpinned" except the paper-value row (the paper prints no potentials, fields or near-field sums).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "p2p_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

CFLAGS = ["-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-std=gnu11"]


def build(force: bool = False) -> str:
    """Compile the oracle C library in-tree (gcc; generic x86-64, no -march so it runs on any host)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_LIB)
            p = C.c_void_p
            i64, i32, u32, dbl = C.c_int64, C.c_int, C.c_uint32, C.c_double
            sig = {
                "orc_bin": (i64, [i32, i64, p, dbl, p, p, p]),
                "orc_bits_per_dim": (i32, [i32, p]),
                "orc_morton": (u32, [i32, i32, p]),
                "orc_demorton": (None, [i32, i32, u32, p]),
                "orc_stable_sort": (None, [i64, p, p, p]),
                "orc_box_table": (i64, [i64, p, p, p]),
                "orc_gravity_structs": (i64, [i64, p, dbl, p, p, u32, p, p, p, p, p, p, p, p, p, p]),
                "orc_gravity_red": (None, [i32, i64, p, p, dbl, p, p, u32, p, p, p, p, p, p, p, p]),
                "orc_gravity_eval_redundant": (None, [i32, i64, p, dbl, p, p, p, p, p, p, p, p, p, p, dbl, p, p]),
                "orc_gravity_eval_indexed": (None, [i64, p, p, dbl, p, u32, p, p, p, p, p, p, dbl, p, p]),
                "orc_gravity_eval_indexed_boxes": (None, [i64, p, p, p, dbl, p, u32, p, p, p, p, p, p, dbl, p, p]),
                "orc_gravity_brute": (i64, [i64, p, p, dbl, p, p, u32, dbl, p, p]),
                "orc_gravity_pairrec": (None, [i32, i64, p, p, dbl, p, p, u32, p, p, p, p, p, p, p, p]),
                "orc_gravity_eval_pairrec": (None, [i32, i64, p, p, p, p, p, p, p, dbl, p, p, p]),
                "orc_helm_weight": (None, [dbl, dbl, dbl, p, p]),
                "orc_helm_table": (None, [i32, dbl, dbl, p]),
                "orc_helm_structs": (i64, [i64, p, dbl, p, p, i32, p, p, p, p, p, p, p]),
                "orc_helm_eval_table": (None, [i64, i32, p, p, p, p, p, p]),
                "orc_helm_dense": (i64, [i64, p, p, dbl, p, p, dbl, dbl, p]),
                "orc_set_threads": (i32, [i32]),
            }
            for name, (res, args) in sig.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


class OutOfDomain(ValueError):
    pass


class Unsupported(ValueError):
    pass


# ------------------------------------------------------------------------------------------------
# primitives (exposed so the pins can test them one by one)
# ------------------------------------------------------------------------------------------------
def morton(dim: int, nb: int, coords) -> int:
    c = np.ascontiguousarray(np.asarray(coords, dtype=np.int32))
    return int(lib().orc_morton(dim, nb, _p(c)))


def demorton(dim: int, nb: int, key: int):
    c = np.zeros(dim, dtype=np.int32)
    lib().orc_demorton(dim, nb, int(key), _p(c))
    return tuple(int(v) for v in c)


def bits_per_dim(nbox) -> int:
    nb = np.ascontiguousarray(np.asarray(nbox, dtype=np.int32))
    return int(lib().orc_bits_per_dim(len(nbox), _p(nb)))


def bin_positions(pos, h, lo, nbox) -> np.ndarray:
    pos = _f64(pos)
    n, dim = pos.shape
    ib = np.zeros((n, dim), dtype=np.int32)
    lo_ = _f64(lo)
    nb = np.ascontiguousarray(np.asarray(nbox, dtype=np.int32))
    bad = lib().orc_bin(dim, n, _p(pos), float(h), _p(lo_), _p(nb), _p(ib))
    if bad >= 0:
        raise OutOfDomain(f"particle {bad} outside the domain")
    return ib


def stable_sort(key):
    key = np.ascontiguousarray(np.asarray(key, dtype=np.uint32))
    n = key.shape[0]
    skey = np.zeros(n, np.uint32)
    perm = np.zeros(n, np.uint32)
    lib().orc_stable_sort(n, _p(key), _p(skey), _p(perm))
    return skey, perm


# ------------------------------------------------------------------------------------------------
# gravity
# ------------------------------------------------------------------------------------------------
class GravityPlan:
    """All oracle structures for one gravity input (a1..a6), plus the three eval modes."""

    def __init__(self, inp, with_red: bool = True):
        self.inp = inp
        self.prec = 0 if inp.pos.dtype == np.float32 else 1
        self.pos = _f64(inp.pos)            # working precision promoted to fp64 (exact)
        self.mass = _f64(inp.mass)
        self.lo = _f64(inp.lo)
        self.nbox = np.ascontiguousarray(np.asarray(inp.nbox, dtype=np.int32))
        n = self.pos.shape[0]
        L = lib()
        self.key = np.zeros(n, np.uint32)
        self.skey = np.zeros(n, np.uint32)
        self.perm = np.zeros(n, np.uint32)
        bkey = np.zeros(max(n, 1), np.uint32)
        bstart = np.zeros(n + 1, np.uint32)
        nbr_off = np.zeros(n + 1, np.uint32)
        nbr_box = np.zeros(max(27 * n, 1), np.uint32)
        nbr_slot = np.zeros(max(27 * n, 1), np.uint8)
        red_off = np.zeros(n + 1, np.uint64)
        counts = np.zeros(4, np.int64)
        bad = L.orc_gravity_structs(n, _p(self.pos), float(inp.h), _p(self.lo), _p(self.nbox), int(inp.periodic),
                                    _p(self.key), _p(self.skey), _p(self.perm), _p(bkey), _p(bstart), _p(nbr_off),
                                    _p(nbr_box), _p(nbr_slot), _p(red_off), _p(counts))
        if bad >= 0:
            raise OutOfDomain(f"particle {bad} outside the domain")
        B, E, R, I = (int(v) for v in counts)
        self.B, self.n_nbr, self.R, self.I = B, E, R, I
        self.bkey = bkey[:B].copy()
        self.bstart = bstart[:B + 1].copy()
        self.nbr_off = nbr_off[:B + 1].copy()
        self.nbr_box = nbr_box[:E].copy()
        self.nbr_slot = nbr_slot[:E].copy()
        self.red_off = red_off[:B + 1].copy()
        self.red = None
        if with_red:
            self.build_red()

    def build_red(self):
        dt = np.float32 if self.prec == 0 else np.float64
        self.red = np.zeros((max(self.R, 1), 4), dt)
        lib().orc_gravity_red(self.prec, self.B, _p(self.pos), _p(self.mass), float(self.inp.h), _p(self.lo),
                              _p(self.nbox), int(self.inp.periodic), _p(self.perm), _p(self.bkey), _p(self.bstart),
                              _p(self.nbr_off), _p(self.nbr_box), _p(self.nbr_slot), _p(self.red_off), _p(self.red))
        self.red = self.red[:self.R]
        return self.red

    def eval_redundant(self):
        n = self.pos.shape[0]
        phi = np.zeros(n)
        field = np.zeros((n, 3))
        red = self.red if self.R > 0 else np.zeros((1, 4), np.float32 if self.prec == 0 else np.float64)
        lib().orc_gravity_eval_redundant(self.prec, self.B, _p(self.pos), float(self.inp.h), _p(self.lo),
                                         _p(self.nbox), _p(self.perm), _p(self.bkey), _p(self.bstart),
                                         _p(self.nbr_off), _p(self.nbr_box), _p(self.nbr_slot), _p(self.red_off),
                                         _p(np.ascontiguousarray(red)), float(self.inp.eps), _p(phi), _p(field))
        return phi, field

    def eval_indexed(self):
        n = self.pos.shape[0]
        phi = np.zeros(n)
        field = np.zeros((n, 3))
        lib().orc_gravity_eval_indexed(self.B, _p(self.pos), _p(self.mass), float(self.inp.h), _p(self.nbox),
                                       int(self.inp.periodic), _p(self.perm), _p(self.bkey), _p(self.bstart),
                                       _p(self.nbr_off), _p(self.nbr_box), _p(self.nbr_slot), float(self.inp.eps),
                                       _p(phi), _p(field))
        return phi, field


    def build_pairrec(self, records: bool = True):
        """the paper's thread-level pair records, one per CSR entry: [targets of b ;
        sources of k], rebased like red (C11).  Returns (pr_off[E+1], pr[P][4]) -- pr None if not records."""
        off = np.zeros(self.n_nbr + 1, np.uint64)
        L = lib()
        L.orc_gravity_pairrec(self.prec, self.B, _p(self.pos), _p(self.mass), float(self.inp.h), _p(self.lo),
                              _p(self.nbox), int(self.inp.periodic), _p(self.perm), _p(self.bkey), _p(self.bstart),
                              _p(self.nbr_off), _p(self.nbr_box), _p(self.nbr_slot), _p(off), None)
        pr = None
        if records:
            dt = np.float32 if self.prec == 0 else np.float64
            pr = np.zeros((max(int(off[-1]), 1), 4), dt)
            L.orc_gravity_pairrec(self.prec, self.B, _p(self.pos), _p(self.mass), float(self.inp.h), _p(self.lo),
                                  _p(self.nbox), int(self.inp.periodic), _p(self.perm), _p(self.bkey),
                                  _p(self.bstart), _p(self.nbr_off), _p(self.nbr_box), _p(self.nbr_slot), _p(off),
                                  _p(pr))
            pr = pr[:int(off[-1])]
        self.pr_off, self.pr = off, pr
        return off, pr

    def eval_pairrec(self):
        """per-(record, target) partials from the record bytes alone, then the deterministic update (ascending
        record order per target).  Returns (phi, field, partial[T][4])."""
        if getattr(self, "pr", None) is None:
            self.build_pairrec()
        n = self.pos.shape[0]
        nb = np.diff(self.bstart.astype(np.int64))
        T = int((np.diff(self.nbr_off.astype(np.int64)) * nb).sum())
        partial = np.zeros((max(T, 1), 4))
        phi = np.zeros(n)
        field = np.zeros((n, 3))
        pr = self.pr if self.pr.shape[0] > 0 else np.zeros((1, 4), self.pr.dtype)
        lib().orc_gravity_eval_pairrec(self.prec, self.B, _p(self.perm), _p(self.bstart), _p(self.nbr_off),
                                       _p(self.nbr_box), _p(self.nbr_slot), _p(self.pr_off),
                                       _p(np.ascontiguousarray(pr)), float(self.inp.eps), _p(partial), _p(phi),
                                       _p(field))
        return phi, field, partial[:T]

    def eval_indexed_boxes(self, boxes):
        """plain definition (mode ii) for the targets of the listed boxes only; returns (phi, field) arrays of
        full length N with NaN outside the listed boxes"""
        n = self.pos.shape[0]
        phi = np.full(n, np.nan)
        field = np.full((n, 3), np.nan)
        sel = np.ascontiguousarray(np.asarray(boxes, dtype=np.uint32))
        lib().orc_gravity_eval_indexed_boxes(sel.shape[0], _p(sel), _p(self.pos), _p(self.mass), float(self.inp.h),
                                             _p(self.nbox), int(self.inp.periodic), _p(self.perm), _p(self.bkey),
                                             _p(self.bstart), _p(self.nbr_off), _p(self.nbr_box), _p(self.nbr_slot),
                                             float(self.inp.eps), _p(phi), _p(field))
        return phi, field

    def pairs_of_boxes(self, boxes) -> int:
        boxes = np.asarray(boxes, dtype=np.int64)
        nb = np.diff(self.bstart.astype(np.int64))
        nsrc = np.diff(self.red_off.astype(np.int64))
        return int((nb[boxes] * nsrc[boxes]).sum())


def gravity_brute(inp):
    pos = _f64(inp.pos)
    mass = _f64(inp.mass)
    n = pos.shape[0]
    phi = np.zeros(n)
    field = np.zeros((n, 3))
    lo = _f64(inp.lo)
    nb = np.ascontiguousarray(np.asarray(inp.nbox, dtype=np.int32))
    bad = lib().orc_gravity_brute(n, _p(pos), _p(mass), float(inp.h), _p(lo), _p(nb), int(inp.periodic),
                                  float(inp.eps), _p(phi), _p(field))
    if bad >= 0:
        raise OutOfDomain(f"particle {bad} outside the domain")
    return phi, field


# ------------------------------------------------------------------------------------------------
# Helmholtz
# ------------------------------------------------------------------------------------------------
def helm_weight(r: float, delta: float, k: float) -> complex:
    re = C.c_double()
    im = C.c_double()
    lib().orc_helm_weight(float(r), float(delta), float(k), C.byref(re), C.byref(im))
    return complex(re.value, im.value)


def helm_table(t: int, delta: float, k: float) -> np.ndarray:
    P = np.zeros((t, 9 * t), np.complex128)
    lib().orc_helm_table(int(t), float(delta), float(k), _p(P))
    return P


class HelmholtzPlan:
    def __init__(self, inp):
        self.inp = inp
        self.pos = _f64(inp.pos)
        self.x = np.ascontiguousarray(np.asarray(inp.x, dtype=np.complex128))
        self.lo = _f64(inp.lo)
        self.nbox = np.ascontiguousarray(np.asarray(inp.nbox, dtype=np.int32))
        n = self.pos.shape[0]
        self.key = np.zeros(n, np.uint32)
        self.skey = np.zeros(n, np.uint32)
        self.perm = np.zeros(n, np.uint32)
        bkey = np.zeros(max(n, 1), np.uint32)
        bstart = np.zeros(n + 1, np.uint32)
        nbr9 = np.zeros(max(9 * n, 1), np.uint32)
        counts = np.zeros(4, np.int64)
        r = lib().orc_helm_structs(n, _p(self.pos), float(inp.h), _p(self.lo), _p(self.nbox), int(inp.t),
                                   _p(self.key), _p(self.skey), _p(self.perm), _p(bkey), _p(bstart), _p(nbr9),
                                   _p(counts))
        if r == -2:
            raise Unsupported("not a regular t-per-box lattice")
        if r >= 0:
            raise OutOfDomain(f"sample {r} outside the domain")
        self.B = int(counts[0])
        self.bkey = bkey[:self.B].copy()
        self.bstart = bstart[:self.B + 1].copy()
        self.nbr9 = nbr9[:9 * self.B].reshape(self.B, 9).copy()
        self.P = helm_table(inp.t, inp.delta, inp.k)

    @property
    def n_pairs(self) -> int:
        """non-padded interactions t^2 * sum_b |N(b)| (C19)"""
        return int(self.inp.t) ** 2 * int(np.count_nonzero(self.nbr9 != 0xFFFFFFFF))

    def xg(self) -> np.ndarray:
        """the redundant (im2col) buffer Xg[B][9][t], zero segments for missing neighbours"""
        t = self.inp.t
        Xg = np.zeros((self.B, 9, t), np.complex128)
        xs = self.x[self.perm]
        for s in range(9):
            k = self.nbr9[:, s]
            ok = k != 0xFFFFFFFF
            idx = self.bstart[k[ok]][:, None] + np.arange(t)[None, :]
            Xg[ok, s, :] = xs[idx]
        return Xg

    def eval_table(self) -> np.ndarray:
        n = self.pos.shape[0]
        y = np.zeros(n, np.complex128)
        lib().orc_helm_eval_table(self.B, int(self.inp.t), _p(self.P), _p(self.x), _p(self.perm),
                                  _p(self.bstart), _p(np.ascontiguousarray(self.nbr9)), _p(y))
        return y


def helm_dense(inp) -> np.ndarray:
    pos = _f64(inp.pos)
    x = np.ascontiguousarray(np.asarray(inp.x, dtype=np.complex128))
    n = pos.shape[0]
    y = np.zeros(n, np.complex128)
    lo = _f64(inp.lo)
    nb = np.ascontiguousarray(np.asarray(inp.nbox, dtype=np.int32))
    bad = lib().orc_helm_dense(n, _p(pos), _p(x), float(inp.h), _p(lo), _p(nb), float(inp.delta), float(inp.k),
                               _p(y))
    if bad >= 0:
        raise OutOfDomain(f"sample {bad} outside the domain")
    return y


def rel_l2(a, b) -> float:
    a = np.asarray(a, dtype=np.complex128 if np.iscomplexobj(a) or np.iscomplexobj(b) else np.float64).ravel()
    b = np.asarray(b, dtype=a.dtype).ravel()
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def set_threads(n: int) -> int:
    """OpenMP threads of the following oracle calls (timing harness only); returns the count in effect."""
    return int(lib().orc_set_threads(int(n)))
