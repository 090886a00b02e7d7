"""Seeded synthetic input generators shared by the oracle tests, the GPU tests and bench.py.

This module is deliberately independent of both sides of the parity check: it holds NO arithmetic of
the method (no binning, no keys, no neighbour logic, no kernel), only random-number recipes that
produce positions and charges with the shapes and distributions of the paper's workloads
(DESIGN.md "Input recipe").  Every generator uses numpy's PCG64 with an explicit seed,
draws in fp64 and rounds ONCE to the working precision, so the oracle and the CUDA path read the
very same bits.

Workloads (PAPER.md lines cited as P:Lnnn):
  * uniform_per_box  -- exactly k uniform-random particles per box of an n^3 periodic grid
                        (BASELINE configs[0] = C1, configs[3] = C4 density sweep; P:L171-175 Locality trend).
  * plummer          -- Plummer-like clustered sphere, scale radius a = 0.1 L, truncated to the box
                        (PhotoNs-2.0-like irregular distribution; configs[2] = C3).
  * plummer_tiles    -- G Plummer tiles side by side (configs[4] = C5 weak/strong scaling).
  * dbim_lattice     -- regular 2D lattice, sqrt(t) x sqrt(t) cell-centred samples per leaf box,
                        complex CN(0,1) unknowns (DBIM-MLFMA-like; configs[1] = C2).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np


@dataclasses.dataclass
class GravityInput:
    pos: np.ndarray          # [N][3] float32 or float64, C-contiguous
    mass: np.ndarray         # [N] same dtype
    lo: tuple                # domain origin (3 doubles)
    h: float                 # box edge
    nbox: tuple              # boxes per dim (3 ints)
    periodic: int            # bit mask
    eps: float               # softening
    name: str = ""

    @property
    def n(self) -> int:
        return int(self.pos.shape[0])


@dataclasses.dataclass
class HelmholtzInput:
    pos: np.ndarray          # [N][2] float32 sample positions (cell centres)
    x: np.ndarray            # [N] complex64 unknowns
    lo: tuple                # (2 doubles)
    h: float                 # box edge = sqrt(t) * delta
    nbox: tuple              # (2 ints)
    t: int                   # samples per box (perfect square)
    delta: float             # sample spacing
    k: float                 # wavenumber = 2*pi/(10*delta)
    name: str = ""

    @property
    def n(self) -> int:
        return int(self.pos.shape[0])


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(int(seed)))


def _round(a: np.ndarray, dtype) -> np.ndarray:
    return np.ascontiguousarray(a.astype(dtype))


def uniform_per_box(n: int, k: int, seed: int = 0, dtype=np.float32, eps: float = 1e-3,
                    shuffle: bool = True, margin: float = 1e-4) -> GravityInput:
    """Exactly k uniform-random particles in every box of an n x n x n periodic grid on [0,1)^3.

    Offsets inside a box are drawn from U[margin, 1-margin) so that rounding to fp32 never moves a
    point across a box face (the count per box stays exactly k).  Input order is shuffled (particle
    order in a PhotoNs step is arbitrary), masses m ~ U[0.5, 1.5)/N.
    """
    rng = _rng(seed)
    N = n * n * n * k
    h = 1.0 / n
    cells = np.repeat(np.arange(n * n * n, dtype=np.int64), k)
    iz, rem = np.divmod(cells, n * n)
    iy, ix = np.divmod(rem, n)
    u = rng.uniform(margin, 1.0 - margin, size=(N, 3))
    pos = np.stack([(ix + u[:, 0]) * h, (iy + u[:, 1]) * h, (iz + u[:, 2]) * h], axis=1)
    mass = rng.uniform(0.5, 1.5, size=N) / N
    if shuffle:
        p = rng.permutation(N)
        pos, mass = pos[p], mass[p]
    return GravityInput(_round(pos, dtype), _round(mass, dtype), (0.0, 0.0, 0.0), h, (n, n, n), 0b111,
                        eps, f"uniform n={n} k={k} seed={seed}")


def _plummer_points(rng: np.random.Generator, N: int, a: float, center, side: float,
                    margin: float) -> np.ndarray:
    """Plummer sphere radius r = a / sqrt(U^{-2/3} - 1), isotropic, rejected to the cube
    [center - side/2 + 0, center + side/2 - margin)."""
    out = np.empty((0, 3))
    lo = np.asarray(center, dtype=np.float64) - side / 2
    hi = lo + side
    while out.shape[0] < N:
        m = int((N - out.shape[0]) * 1.3) + 64
        u = rng.uniform(1e-12, 1.0, size=m)
        r = a / np.sqrt(u ** (-2.0 / 3.0) - 1.0)
        v = rng.normal(size=(m, 3))
        v /= np.linalg.norm(v, axis=1, keepdims=True)
        p = np.asarray(center) + r[:, None] * v
        ok = np.all((p >= lo) & (p < hi - margin * side), axis=1)
        out = np.concatenate([out, p[ok]], axis=0)
    return out[:N]


def plummer(N: int, n: int, seed: int = 0, dtype=np.float32, eps: float = 1e-3,
            a: float = 0.1) -> GravityInput:
    """Plummer-like clustered distribution in the periodic unit cube with n^3 leaf boxes."""
    rng = _rng(seed)
    pos = _plummer_points(rng, N, a, (0.5, 0.5, 0.5), 1.0, 1e-7)
    mass = rng.uniform(0.5, 1.5, size=N) / N
    return GravityInput(_round(pos, dtype), _round(mass, dtype), (0.0, 0.0, 0.0), 1.0 / n, (n, n, n),
                        0b111, eps, f"plummer N={N} n={n} seed={seed}")


TILE_ARRANGEMENT = {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}


def plummer_tiles(n_per_tile: int, boxes_per_tile: int, tiles: int, seed: int = 0, dtype=np.float32,
                  eps: float = 1e-3, a: float = 0.1, tile_index=None) -> GravityInput:
    """G Plummer tiles (a = 0.1 tile side) arranged 1x1x1 / 2x1x1 / 2x2x1 / 2x2x2 in a periodic domain
    of tile side 1.  Each tile is seeded with seed*1000 + tile so that tile g is the
    same particles whatever the total tile count (weak scaling).  `tile_index` selects one tile only
    (a rank's initial slice)."""
    ax = TILE_ARRANGEMENT[tiles]
    sel = range(tiles) if tile_index is None else [tile_index]
    ps, ms = [], []
    for g in sel:
        rng = _rng(seed * 1000 + g)
        gx, gy, gz = g % ax[0], (g // ax[0]) % ax[1], g // (ax[0] * ax[1])
        c = (gx + 0.5, gy + 0.5, gz + 0.5)
        p = _plummer_points(rng, n_per_tile, a, c, 1.0, 1e-7)
        ps.append(p)
        ms.append(rng.uniform(0.5, 1.5, size=n_per_tile) / (n_per_tile * tiles))
    pos = np.concatenate(ps)
    mass = np.concatenate(ms)
    nb = (boxes_per_tile * ax[0], boxes_per_tile * ax[1], boxes_per_tile * ax[2])
    return GravityInput(_round(pos, dtype), _round(mass, dtype), (0.0, 0.0, 0.0), 1.0 / boxes_per_tile,
                        nb, 0b111, eps, f"plummer_tiles G={tiles} n/tile={n_per_tile} seed={seed}")


def random_gravity(N: int, n: int, seed: int = 0, dtype=np.float32, eps: float = 1e-3,
                   periodic: int = 0b111, nbox=None, lo=(0.0, 0.0, 0.0), h=None) -> GravityInput:
    """Plain uniform-random particles (ragged occupancy, empty boxes possible) for parity sweeps."""
    rng = _rng(seed)
    nb = tuple(nbox) if nbox is not None else (n, n, n)
    hh = (1.0 / max(nb)) if h is None else h
    ext = np.array([nb[0] * hh, nb[1] * hh, nb[2] * hh])
    pos = np.asarray(lo) + rng.uniform(0.0, 1.0, size=(N, 3)) * ext * (1.0 - 1e-7)
    mass = rng.uniform(0.5, 1.5, size=N) / max(N, 1)
    return GravityInput(_round(pos, dtype), _round(mass, dtype), tuple(lo), hh, nb, periodic, eps,
                        f"random N={N} nbox={nb} seed={seed}")


def dbim_lattice(n: int, t: int, seed: int = 0, delta: float = 1.0, holes=None) -> HelmholtzInput:
    """Regular 2D DBIM-like mesh: n x n leaf boxes, sqrt(t) x sqrt(t) cell-centred samples per box,
    sample spacing delta, k = 2 pi / (10 delta) (10 samples per wavelength),
    unknowns x ~ CN(0,1) ("Input vectors are generated randomly").  Samples are listed in
    global row-major order (y slow, x fast).  `holes` = optional list of (bx, by) boxes left empty
    (exercises missing-neighbour zero segments)."""
    rng = _rng(seed)
    st = int(round(math.sqrt(t)))
    assert st * st == t
    m = n * st
    gy, gx = np.divmod(np.arange(m * m, dtype=np.int64), m)
    keep = np.ones(m * m, dtype=bool)
    if holes:
        for (bx, by) in holes:
            keep &= ~((gx // st == bx) & (gy // st == by))
    gx, gy = gx[keep], gy[keep]
    pos = np.stack([(gx + 0.5) * delta, (gy + 0.5) * delta], axis=1)
    N = pos.shape[0]
    x = (rng.normal(size=N) + 1j * rng.normal(size=N)) / math.sqrt(2.0)
    return HelmholtzInput(_round(pos, np.float32), _round(x, np.complex64), (0.0, 0.0), st * delta, (n, n), t,
                          delta, 2.0 * math.pi / (10.0 * delta), f"dbim n={n} t={t} seed={seed}")


# Named configurations of BASELINE.json.
def config(name: str, seed: int = 0, dtype=np.float32):
    if name == "c1":
        return uniform_per_box(4, 16, seed, dtype)
    if name == "c2a":
        return dbim_lattice(256, 16, seed)
    if name == "c2b":
        return dbim_lattice(256, 64, seed)
    if name == "c3":
        return plummer(1_000_000, 128, seed, dtype)
    if name == "c3dense":
        return plummer(1_000_000, 64, seed, dtype)
    if name.startswith("c4-"):
        k = int(name.split("-")[1])
        n = {8: 108, 16: 85, 32: 68, 64: 54, 128: 43}[k]
        return uniform_per_box(n, k, seed, dtype)
    if name == "c5w":
        return plummer_tiles(12_500_000, 256, 1, seed, dtype)
    if name.startswith("c5w-"):
        g = int(name.split("-")[1])
        return plummer_tiles(12_500_000, 256, g, seed, dtype)
    if name == "c5s":
        return plummer_tiles(12_500_000, 256, 8, seed, dtype)
    raise KeyError(name)
