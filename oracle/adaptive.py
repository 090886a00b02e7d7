"""Adaptive leaves -- TEST INFRASTRUCTURE ONLY, like the rest of oracle/ (only tests/,
smoke() and bench.py's CPU legs may import it; it never imports the product).

Plain numpy definitions for small inputs (no blocking, no fusion), fp64, written from the paper's irregular
binary tree ("an irregular binary MLFMA tree ... with tree rebuilding at each time step"; "The
binary tree structure is highly irregular, with varying depths"), PhotoNs' clustering threshold t (P:L344,
P:L400 Fig 8) and SPEC's ledger for what the paper leaves open.  Readings:

C22 tree.  Periodic cube [lo, lo + L)^3 on a finest grid of n = 2^m boxes per dimension (h = L / n, binning C6,
    Morton keys C7 with 3m bits).  Binary LONGEST-AXIS MIDPOINT splits, ties broken z, y, x -- exactly the Morton
    key's bit order, so a cell is a key prefix of length l (s_z = ceil(l/3), s_y = floor((l+1)/3), s_x = floor(l/3)
    halvings per dimension).  A cell is split while it holds more than t particles or while l < min_bits (default
    9: cells <= L/8 per dimension, so periodic images are unique); finest cells (l = 3m) are leaves whatever their
    count; empty cells are no leaves.  SPEC splits at the median; the midpoint keeps cells aligned to the Morton
    grid (the GPU builds them from the sorted keys).  Leaves are listed in Morton (prefix) order; each holds one
    contiguous run of the key-sorted particles.
C23 adjacency.  B is a neighbour of A under the periodic image S (in units of L) when B + S overlaps (positive
    volume) D(A) = A dilated by one extent of A in each dimension (SPEC: "dilation by one target-box extent"),
    then the symmetric closure is taken (SPEC: "symmetric closure enforced afterward"): the list of A is
    {(B, S): B + S overlaps D(A)} u {(B, S): A - S overlaps D(B)}.  Equal-size leaves reduce to the 27-box stencil
    (C4).  Entries are ordered by (B, image code 9(s_z+1) + 3(s_y+1) + (s_x+1)).
C24 records and eval.  As C11 / C1 with the entry's image S and the TARGET leaf's origin
    o_d = fma(c_d, w_d, lo_d), w_d = L / 2^{s_d} (c_d = the leaf's cell index along d): red = {fl_p(((double)x_j +
    S_d L) - o_d), m_j}; phi_i = -sum_{(j, S) != (i, 0)} m_j (r^2 + eps^2)^{-1/2}, a_i = sum m_j d (r^2 + eps^2)^{-3/2}
    over the sources of the entries of i's leaf.
"""
from __future__ import annotations

import numpy as np

from . import bin_positions


def _interleave(ib: np.ndarray, m: int) -> np.ndarray:
    """3D Morton keys (C7: bit 3k = x_k, 3k+1 = y_k, 3k+2 = z_k) of integer box coordinates, a plain bit loop"""
    key = np.zeros(ib.shape[0], np.int64)
    for k in range(m):
        for d in range(3):
            key |= ((ib[:, d].astype(np.int64) >> k) & 1) << (3 * k + d)
    return key


def halvings(l: int):
    """(s_x, s_y, s_z): halvings per dimension of a cell given by an l-bit key prefix (z first, then y, x)"""
    return (l // 3, (l + 1) // 3, (l + 2) // 3)


class AdaptiveTree:
    """Leaves, closed neighbour lists, redundant records and the plain-definition eval for one input."""

    def __init__(self, inp, t: int, min_bits: int = 9):
        n = int(inp.nbox[0])
        assert tuple(inp.nbox) == (n, n, n) and n & (n - 1) == 0 and inp.periodic == 0b111
        self.inp, self.t, self.n = inp, int(t), n
        self.m = n.bit_length() - 1
        self.min_bits = min(int(min_bits), 3 * self.m)
        self.L = float(np.float64(n) * np.float64(inp.h))   # IEEE product (C5)
        self.lo = np.asarray(inp.lo, np.float64)
        self.pos = inp.pos.astype(np.float64)
        self.mass = inp.mass.astype(np.float64)
        self.ib = bin_positions(inp.pos, inp.h, inp.lo, inp.nbox).astype(np.int64)
        self.key = _interleave(self.ib, self.m)
        self.perm = np.argsort(self.key, kind="stable")      # sorted slot -> input index (ties: input order)
        self.skey = self.key[self.perm]
        self.leaves = self._build()                          # [(l, prefix, start, count)] in Morton order
        self.nleaf = len(self.leaves)
        self.leaf_of = np.zeros(len(self.key), np.int64)     # input index -> leaf
        for a, (_, _, s, c) in enumerate(self.leaves):
            self.leaf_of[self.perm[s:s + c]] = a
        # leaf boxes in finest-box units (exact integers): lower corner and width per dimension
        self.lo_i = np.zeros((self.nleaf, 3), np.int64)
        self.w_i = np.zeros((self.nleaf, 3), np.int64)
        for a, (l, _, s, _) in enumerate(self.leaves):
            sh = halvings(l)
            first = self.ib[self.perm[s]]
            for d in range(3):
                w = n >> sh[d]
                self.w_i[a, d] = w
                self.lo_i[a, d] = (first[d] // w) * w

    # ---- C22: top-down midpoint splits on the sorted keys ----
    def _build(self):
        out = []
        bits = 3 * self.m

        def rec(l, prefix, s, e):
            if e == s:
                return
            if l == bits or (l >= self.min_bits and e - s <= self.t):
                out.append((l, prefix, s, e - s))
                return
            child = (prefix << 1) | 1                           # first key of the upper half: prefix.1 000...
            mid = s + int(np.searchsorted(self.skey[s:e], child << (bits - l - 1), side="left"))
            rec(l + 1, prefix << 1, s, mid)
            rec(l + 1, child, mid, e)

        rec(0, 0, 0, len(self.skey))
        return out

    # ---- C23: the definition, all leaf pairs ----
    def _overlap0(self):
        """ov[a][code] = boolean array over B: B + S(code) overlaps D(A) (positive volume), exact integers"""
        n = self.n
        lo, w = self.lo_i, self.w_i
        ov = np.zeros((self.nleaf, 27, self.nleaf), bool)
        for code in range(27):
            S = np.array([code % 3 - 1, code // 3 % 3 - 1, code // 9 - 1], np.int64) * n
            ok = np.ones((self.nleaf, self.nleaf), bool)
            for d in range(3):
                dlo = (lo[:, d] - w[:, d])[:, None]                 # D(A) = [lo - w, lo + 2w)
                dhi = (lo[:, d] + 2 * w[:, d])[:, None]
                blo = (lo[:, d] + S[d])[None, :]
                bhi = (lo[:, d] + w[:, d] + S[d])[None, :]
                ok &= (blo < dhi) & (bhi > dlo)
            ov[:, code, :] = ok
        return ov

    def neighbours(self):
        """closed lists: nbr[a] = sorted [(b, code)] with (b, S) in N0(a) or (a, -S) in N0(b)"""
        if getattr(self, "_nbr", None) is not None:
            return self._nbr
        ov = self._overlap0()
        closed = ov | ov[:, ::-1, :].transpose(2, 1, 0)      # (a, code, b) or (b, 26 - code, a)
        self._nbr = []
        for a in range(self.nleaf):
            c, b = np.nonzero(closed[a])
            o = np.lexsort((c, b))                              # by (b, code)
            self._nbr.append([(int(x), int(y)) for x, y in zip(b[o], c[o])])
        return self._nbr

    # ---- a list construction by range lookups (the GPU's first version), pinned against the definition; the GPU now
    # ---- builds the same lists as dilation + its transpose (k_adaptive.cu), tested against neighbours() directly ----
    def neighbours_by_ranges(self):
        """nbr(B) = {leaves of level >= l_B inside B's 27 same-shape cells} u {coarser leaves A with A one of the
        27 cells around B's level-l_A ancestor}; same order as neighbours()"""
        index = {}                                             # (l, cell coords) -> leaf
        for a, (l, _, _, _) in enumerate(self.leaves):
            index[(l, tuple(int(v) for v in self.lo_i[a] // self.w_i[a]))] = a

        def around(cell, sh):
            """the 27 cells around `cell` at halvings sh: (wrapped cell, image code)"""
            cells = 1 << np.array(sh)
            for code in range(27):
                cc = cell + np.array([code % 3 - 1, code // 3 % 3 - 1, code // 9 - 1])
                img = np.where(cc < 0, -1, np.where(cc >= cells, 1, 0))
                yield cc - img * cells, int(9 * (img[2] + 1) + 3 * (img[1] + 1) + (img[0] + 1))

        levels = np.array([l for l, _, _, _ in self.leaves])
        out = []
        for b, (lb, _, _, _) in enumerate(self.leaves):
            res = set()
            wb = self.w_i[b]
            for cc, code in around(self.lo_i[b] // wb, halvings(lb)):      # dilation: finer-or-equal leaves
                x0, x1 = cc * wb, (cc + 1) * wb
                inside = (levels >= lb) & np.all(self.lo_i >= x0, axis=1) & np.all(self.lo_i + self.w_i <= x1, axis=1)
                res.update((int(a), code) for a in np.nonzero(inside)[0])
            for la in range(lb):                                          # closure: coarser leaves
                sh = halvings(la)
                w = self.n >> np.array(sh)
                for cc, code in around(self.lo_i[b] // w, sh):
                    a = index.get((la, tuple(int(v) for v in cc)))
                    if a is not None:
                        res.add((a, code))
            out.append(sorted(res))
        return out

    # ---- C24 ----
    def origin(self, a: int) -> np.ndarray:
        """o_d = fma(c_d, w_d, lo_d), w_d = L / 2^s_d (exact scaling), one rounding (exact rationals)"""
        w = self.L / (self.n // self.w_i[a]).astype(np.float64)
        c = (self.lo_i[a] // self.w_i[a]).astype(np.float64)
        return np.array([_fma(float(c[d]), float(w[d]), float(self.lo[d])) for d in range(3)])

    def red(self, prec=np.float32):
        """redundant records of every target leaf in leaf order, entries in list order"""
        out = []
        nbr = self.neighbours()
        for a in range(self.nleaf):
            o = self.origin(a)
            for b, code in nbr[a]:
                S = np.array([code % 3 - 1, code // 3 % 3 - 1, code // 9 - 1], np.float64) * self.L
                _, _, s, c = self.leaves[b]
                idx = self.perm[s:s + c]
                x = ((self.pos[idx] + S) - o).astype(prec)
                out.append(np.concatenate([x, self.mass[idx, None].astype(prec)], axis=1))
        return np.concatenate(out) if out else np.zeros((0, 4), prec)

    def eval(self, eps: float):
        """phi, field from the closed lists (plain definition, fp64, d = (x_j + S) - x_i from the inputs)"""
        N = len(self.key)
        phi, field = np.zeros(N), np.zeros((N, 3))
        e2 = eps * eps
        nbr = self.neighbours()
        for a in range(self.nleaf):
            _, _, s, c = self.leaves[a]
            ti = self.perm[s:s + c]
            src, sm, self_mask = [], [], []
            for b, code in nbr[a]:
                S = np.array([code % 3 - 1, code // 3 % 3 - 1, code // 9 - 1], np.float64) * self.L
                _, _, sb, cb = self.leaves[b]
                sj = self.perm[sb:sb + cb]
                src.append(self.pos[sj] + S)
                sm.append(self.mass[sj])
                self_mask.append(sj[None, :] == ti[:, None] if (b == a and code == 13) else
                                 np.zeros((len(ti), len(sj)), bool))
            X, M, SELF = np.concatenate(src), np.concatenate(sm), np.concatenate(self_mask, axis=1)
            d = X[None, :, :] - self.pos[ti][:, None, :]
            r2 = (d * d).sum(axis=2) + e2
            ri = 1.0 / np.sqrt(r2)
            phi[ti] = -np.where(SELF, 0.0, M[None, :] * ri).sum(axis=1)
            field[ti] = ((M[None, :] * ri ** 3)[:, :, None] * d).sum(axis=1)
        return phi, field

    def pair_count(self) -> int:
        nbr = self.neighbours()
        return sum(self.leaves[a][3] * sum(self.leaves[b][3] for b, _ in nbr[a]) for a in range(self.nleaf))


def _fma(a: float, b: float, c: float) -> float:
    """a * b + c with ONE rounding: exact rational arithmetic, Fraction -> float rounds to nearest even"""
    from fractions import Fraction
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def brute(tree: AdaptiveTree, eps: float):
    """all particle pairs with the closed adjacency PREDICATE evaluated directly from the leaf boxes (no lists):
    j (image S) acts on i iff leaf(j) + S overlaps D(leaf(i)) or leaf(i) - S overlaps D(leaf(j))"""
    n = tree.n
    N = len(tree.key)
    A, Bl = tree.leaf_of[:, None], tree.leaf_of[None, :]
    phi, field = np.zeros(N), np.zeros((N, 3))
    e2 = eps * eps
    for code in range(27):
        Sv = np.array([code % 3 - 1, code // 3 % 3 - 1, code // 9 - 1], np.int64)
        fwd = np.ones((N, N), bool)
        bwd = np.ones((N, N), bool)
        for d in range(3):
            alo, aw = tree.lo_i[A, d], tree.w_i[A, d]
            blo, bw = tree.lo_i[Bl, d], tree.w_i[Bl, d]
            S = Sv[d] * n
            fwd &= (blo + S < alo + 2 * aw) & (blo + bw + S > alo - aw)      # B + S overlaps D(A)
            bwd &= (alo - S < blo + 2 * bw) & (alo + aw - S > blo - bw)      # A - S overlaps D(B)
        act = fwd | bwd
        if code == 13:
            np.fill_diagonal(act, False)                                     # the self pair (C3)
        if not act.any():
            continue
        Sx = Sv.astype(np.float64) * tree.L
        d = (tree.pos[None, :, :] + Sx) - tree.pos[:, None, :]
        r2 = (d * d).sum(axis=2) + e2
        ri = np.where(act, 1.0 / np.sqrt(r2), 0.0)
        phi -= (tree.mass[None, :] * ri).sum(axis=1)
        field += ((tree.mass[None, :] * ri ** 3)[:, :, None] * d).sum(axis=1)
    return phi, field


def neighbours_of(tree: AdaptiveTree, a: int):
    """the closed list of ONE leaf straight from the definition (vectorised over the other leaves): for full-size
    sampled checks where the all-pairs lists are out of reach"""
    n = tree.n
    lo, w = tree.lo_i, tree.w_i
    out = []
    for code in range(27):
        S = np.array([code % 3 - 1, code // 3 % 3 - 1, code // 9 - 1], np.int64) * n
        fwd = np.ones(tree.nleaf, bool)   # B + S overlaps D(a)
        bwd = np.ones(tree.nleaf, bool)   # a - S overlaps D(B)
        for d in range(3):
            fwd &= (lo[:, d] + S[d] < lo[a, d] + 2 * w[a, d]) & (lo[:, d] + w[:, d] + S[d] > lo[a, d] - w[a, d])
            bwd &= (lo[a, d] - S[d] < lo[:, d] + 2 * w[:, d]) & (lo[a, d] + w[a, d] - S[d] > lo[:, d] - w[:, d])
        out += [(int(b), code) for b in np.nonzero(fwd | bwd)[0]]
    return sorted(out)


def eval_leaf(tree: AdaptiveTree, a: int, eps: float, nbr=None):
    """phi, field of leaf a's targets (plain definition, fp64) from its closed list; returns (input indices, phi,
    field)"""
    nbr = neighbours_of(tree, a) if nbr is None else nbr
    _, _, s, c = tree.leaves[a]
    ti = tree.perm[s:s + c]
    X, M, SELF = [], [], []
    for b, code in nbr:
        S = np.array([code % 3 - 1, code // 3 % 3 - 1, code // 9 - 1], np.float64) * tree.L
        _, _, sb, cb = tree.leaves[b]
        sj = tree.perm[sb:sb + cb]
        X.append(tree.pos[sj] + S)
        M.append(tree.mass[sj])
        SELF.append(sj[None, :] == ti[:, None] if (b == a and code == 13) else np.zeros((len(ti), len(sj)), bool))
    X, M, SELF = np.concatenate(X), np.concatenate(M), np.concatenate(SELF, axis=1)
    d = X[None, :, :] - tree.pos[ti][:, None, :]
    ri = 1.0 / np.sqrt((d * d).sum(axis=2) + eps * eps)
    phi = -np.where(SELF, 0.0, M[None, :] * ri).sum(axis=1)
    field = ((M[None, :] * ri ** 3)[:, :, None] * d).sum(axis=1)
    return ti, phi, field


def brute_pairs(tree: AdaptiveTree) -> int:
    """number of acting (i, j, S) triples of the closed adjacency predicate, self pair excluded (see brute)"""
    n = tree.n
    A, Bl = tree.leaf_of[:, None], tree.leaf_of[None, :]
    tot = 0
    for code in range(27):
        Sv = np.array([code % 3 - 1, code // 3 % 3 - 1, code // 9 - 1], np.int64)
        fwd = np.ones((len(tree.key), len(tree.key)), bool)
        bwd = np.ones_like(fwd)
        for d in range(3):
            alo, aw = tree.lo_i[A, d], tree.w_i[A, d]
            blo, bw = tree.lo_i[Bl, d], tree.w_i[Bl, d]
            S = Sv[d] * n
            fwd &= (blo + S < alo + 2 * aw) & (blo + bw + S > alo - aw)
            bwd &= (alo - S < blo + 2 * bw) & (alo + aw - S > blo - bw)
        act = fwd | bwd
        if code == 13:
            np.fill_diagonal(act, False)
        tot += int(act.sum())
    return tot


def leaf_count_bottom_up(key: np.ndarray, m: int, t: int, min_bits: int) -> int:
    """independent recount ("leaf count equals an independent recursive-count oracle"): a particle's
    leaf is the SHORTEST prefix l >= min_bits whose cell holds <= t particles (or l = 3m); leaves = distinct
    (l, prefix) pairs"""
    bits = 3 * m
    leaf_l = np.full(len(key), bits, np.int64)
    for l in range(bits, min(min_bits, bits) - 1, -1):
        pre = key >> (bits - l)
        _, inv, cnt = np.unique(pre, return_inverse=True, return_counts=True)
        small = cnt[inv] <= t
        leaf_l = np.where(small, l, leaf_l)
    pairs = {(int(l), int(k >> (bits - l))) for l, k in zip(leaf_l, key)}
    return len(pairs)
