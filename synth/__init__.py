"""Seeded synthetic particle clouds shared by the oracle tests, the CUDA parity
tests and bench.py.

This module holds NO arithmetic of the method (no cell index, no binning, no
pair interaction).  It only draws the inputs: fp32 positions in the box and
fp32 per-particle values, with the shapes of the paper's workloads
(§7.1: uniform particles, d^3 grids, 1/10/100 particles per
cell, single precision) and of BASELINE.json's configs.  Both the oracle and
the GPU path consume exactly the bytes returned here.

Recipe:
  * rng = numpy.random.Generator(PCG64(seed)), seed = 240616091 + config index
  * positions: rng.random((3, n), dtype=float32) * box extent + origin.  For
    every shipped config the extent is a power of two, so the scaling is exact.
  * values: q = rng.uniform(0.5, 1.5, n).astype(float32)
  * clustered: 75 % in 32 isotropic Gaussian blobs (sigma_b = 0.04, centres
    U[0.15, 0.85]^3, equal weights) + 25 % uniform, wrapped mod 1 and clamped
    below 1 (SURVEY.md §8(d) configs[3]).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

SEED_BASE = 240616091


@dataclasses.dataclass(frozen=True)
class Grid:
    """Cell grid: origin, cell width w, dims (Nx, Ny, Nz), cutoff r_c, kernel width sigma.

    Linearisation is X-fastest (§5.1): lin = cx + Nx*(cy + Ny*cz).
    """
    dims: tuple
    w: float
    origin: tuple = (0.0, 0.0, 0.0)
    rc: float | None = None
    sigma: float | None = None
    lj_r: float | None = None      # Lennard-Jones reference length r of Eq. (1) (default r_c)
    lj_eps: float | None = None    # softening (default r_c / 20)
    lj_e0: float = 1.0             # E_0

    @property
    def r_c(self) -> float:
        return float(self.w if self.rc is None else self.rc)

    @property
    def lj_ref(self) -> float:
        return float(self.r_c if self.lj_r is None else self.lj_r)

    @property
    def lj_soft(self) -> float:
        return float(self.r_c / 20.0 if self.lj_eps is None else self.lj_eps)

    @property
    def sig(self) -> float:
        return float(self.r_c / 3.0 if self.sigma is None else self.sigma)

    @property
    def ncells(self) -> int:
        return int(self.dims[0]) * int(self.dims[1]) * int(self.dims[2])

    @property
    def extent(self) -> tuple:
        return tuple(float(d) * float(self.w) for d in self.dims)


@dataclasses.dataclass
class Cloud:
    grid: Grid
    x: np.ndarray
    y: np.ndarray
    z: np.ndarray
    q: np.ndarray
    name: str = ""

    @property
    def n(self) -> int:
        return int(self.x.shape[0])


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def charges(rng: np.random.Generator, n: int, kind: str = "pos") -> np.ndarray:
    if kind == "pos":
        return rng.uniform(0.5, 1.5, n).astype(np.float32)
    if kind == "signed":
        return rng.uniform(-1.0, 1.0, n).astype(np.float32)
    if kind == "ones":
        return np.ones(n, dtype=np.float32)
    raise ValueError(kind)


def uniform(n: int, grid: Grid, seed: int, qkind: str = "pos") -> Cloud:
    rng = _rng(seed)
    u = rng.random((3, n), dtype=np.float32)
    ext = grid.extent
    o = grid.origin
    x = (u[0] * np.float32(ext[0]) + np.float32(o[0])).astype(np.float32)
    y = (u[1] * np.float32(ext[1]) + np.float32(o[1])).astype(np.float32)
    z = (u[2] * np.float32(ext[2]) + np.float32(o[2])).astype(np.float32)
    q = charges(rng, n, qkind)
    return Cloud(grid, x, y, z, q, name=f"uniform{n}")


def clustered(n: int, grid: Grid, seed: int, nblobs: int = 32, sigma_b: float = 0.04,
              frac: float = 0.75, qkind: str = "pos") -> Cloud:
    """configs[3]: Gaussian blobs in the unit box (assumes extent 1 in every axis)."""
    rng = _rng(seed)
    nb = int(round(frac * n))
    centres = rng.uniform(0.15, 0.85, (nblobs, 3))
    which = rng.integers(0, nblobs, nb)
    pts_b = centres[which] + rng.normal(0.0, sigma_b, (nb, 3))
    pts_u = rng.random((n - nb, 3))
    pts = np.concatenate([pts_b, pts_u], axis=0)
    pts = np.mod(pts, 1.0)
    pts = pts.astype(np.float32)
    below_one = np.nextafter(np.float32(1.0), np.float32(0.0))
    pts = np.minimum(pts, below_one)
    perm = rng.permutation(n)
    pts = pts[perm]
    ext = grid.extent
    x = (pts[:, 0] * np.float32(ext[0]) + np.float32(grid.origin[0])).astype(np.float32)
    y = (pts[:, 1] * np.float32(ext[1]) + np.float32(grid.origin[1])).astype(np.float32)
    z = (pts[:, 2] * np.float32(ext[2]) + np.float32(grid.origin[2])).astype(np.float32)
    q = charges(rng, n, qkind)
    return Cloud(grid, np.ascontiguousarray(x), np.ascontiguousarray(y), np.ascontiguousarray(z), q,
                 name=f"clustered{n}")


def lattice(d: int, qkind: str = "ones", seed: int = 0) -> Cloud:
    """C14 dyadic lattice: d^3 cells of width w = 1/d (d a power of two), a simple
    cubic lattice of spacing a = w/2 (8 points per cell) at (k + 1/2) a, r_c = 2a,
    sigma = r_c/3.  Every coordinate is dyadic, so r^2 is exact in fp32 and fp64."""
    w = 1.0 / d
    a = w / 2.0
    k = (np.arange(2 * d, dtype=np.float64) + 0.5) * a
    X, Y, Z = np.meshgrid(k, k, k, indexing="ij")
    x = X.ravel().astype(np.float32)
    y = Y.ravel().astype(np.float32)
    z = Z.ravel().astype(np.float32)
    grid = Grid(dims=(d, d, d), w=w, rc=2 * a)
    q = charges(_rng(seed), x.shape[0], qkind)
    return Cloud(grid, x, y, z, q, name=f"lattice{d}")


def hand_2x3(variant: str = "A") -> Cloud:
    """C12: the hand-worked 2x3x1 example in the spirit of Fig. 1.
    Origin 0, w = r_c = 1, z = 1/2, q_i = i + 1, dyadic coordinates."""
    pts = [(13 / 8, 5 / 2), (1 / 8, 5 / 4), (1 / 4, 1 / 4), (1 / 4, 9 / 4), (3 / 2, 1 / 2),
           (7 / 8, 15 / 8), (3 / 4, 7 / 8), (3 / 4, 11 / 4), (1 / 2, 3 / 2)]
    if variant == "B":
        pts[1] = (1 / 4, 5 / 4)
    x = np.array([p[0] for p in pts], dtype=np.float32)
    y = np.array([p[1] for p in pts], dtype=np.float32)
    z = np.full(9, 0.5, dtype=np.float32)
    q = np.arange(1, 10, dtype=np.float32)
    grid = Grid(dims=(2, 3, 1), w=1.0, rc=1.0)
    return Cloud(grid, x, y, z, q, name=f"hand2x3{variant}")


# --------------------------------------------------------------------------------------
# BASELINE.json configs.  configs[k] -> seed SEED_BASE + k.
# --------------------------------------------------------------------------------------

def config_grid(name: str) -> Grid:
    if name == "c0":
        return Grid(dims=(16, 16, 16), w=1 / 16)
    if name == "c1":
        return Grid(dims=(64, 64, 64), w=1 / 64)
    if name == "c3":
        return Grid(dims=(128, 128, 128), w=1 / 128)
    if name == "c4":
        return Grid(dims=(256, 256, 256), w=1 / 256)
    if name.startswith("c2_ppc"):
        ppc = int(name[len("c2_ppc"):])
        # 2^24 particles, cubic cells w = 2^-k, box extents powers of two.
        table = {1: (256, 256, 256, 256), 2: (256, 256, 128, 256), 4: (256, 128, 128, 256),
                 8: (128, 128, 128, 128), 16: (128, 128, 64, 128), 32: (128, 64, 64, 128),
                 64: (64, 64, 64, 64)}
        nx, ny, nz, inv = table[ppc]
        return Grid(dims=(nx, ny, nz), w=1.0 / inv)
    raise KeyError(name)


CONFIG_N = {"c0": 4096, "c1": 1 << 21, "c3": 1 << 24, "c4": 1 << 27}
CONFIG_INDEX = {"c0": 0, "c1": 1, "c3": 3, "c4": 4}


def make_config(name: str, n: int | None = None, seed_offset: int = 0, qkind: str = "pos") -> Cloud:
    grid = config_grid(name)
    if name.startswith("c2_ppc"):
        idx, nn = 2, 1 << 24
    else:
        idx, nn = CONFIG_INDEX[name], CONFIG_N[name]
    if n is not None:
        nn = n
    seed = SEED_BASE + idx + seed_offset
    if name == "c3":
        c = clustered(nn, grid, seed, qkind=qkind)
    else:
        c = uniform(nn, grid, seed, qkind=qkind)
    c.name = name
    return c


def scaled_uniform(ppc: float, dims: tuple, seed: int, qkind: str = "pos") -> Cloud:
    """Uniform cloud with ~ppc particles per cell on a grid of cubic cells of width 1/max(dims)
    rounded to a power of two (keeps every scaling exact)."""
    m = max(dims)
    inv = 1 << int(math.ceil(math.log2(m)))
    grid = Grid(dims=tuple(int(d) for d in dims), w=1.0 / inv)
    n = int(round(ppc * grid.ncells))
    return uniform(n, grid, seed, qkind=qkind)


def slab_uniform(ppc: float, slab_dims: tuple, rank: int, nranks: int, seed: int, qkind: str = "pos") -> Cloud:
    """Rank `rank`'s share of a weak-scaling X-slab workload: the global grid is
    (slab_dims[0] * nranks, slab_dims[1], slab_dims[2]) cells of width w = 2^-ceil(log2(max(slab_dims))),
    and this rank draws ~ppc particles per cell uniformly inside its own slab
    [rank * Lx * w, (rank + 1) * Lx * w) (independent stream per rank, so the union is a uniform cloud).
    w is a power of two, so the slab faces are exact in fp32 and every particle's cell lies in the slab."""
    lx, ny, nz = (int(d) for d in slab_dims)
    m = max(lx, ny, nz)
    w = 1.0 / (1 << int(math.ceil(math.log2(m))))
    grid = Grid(dims=(lx * nranks, ny, nz), w=w)
    n = int(round(ppc * lx * ny * nz))
    rng = _rng(seed + 7919 * rank)
    u = rng.random((3, n))
    lo, hi = rank * lx * w, (rank + 1) * lx * w
    ext = grid.extent

    def place(v, a, b):
        return np.clip((a + v * (b - a)).astype(np.float32), np.float32(a), np.nextafter(np.float32(b), np.float32(0)))

    x = place(u[0], lo, hi)
    y = place(u[1], 0.0, ext[1])
    z = place(u[2], 0.0, ext[2])
    q = charges(rng, n, qkind)
    return Cloud(grid, x, y, z, q, name=f"slab{rank}of{nranks}")
