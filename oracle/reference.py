"""ORACLE (test infrastructure only; see oracle/__init__.py).

numpy fp64 oracle of the hot path of arXiv 2406.16091, written from the paper:

  PAPER.md:49-51  (§2)  the result: for every i, interactions with all j != i
                        such that r_ij < r_c, through a kernel K(r_ij).
  PAPER.md:58-65  (§2)  the pipeline: cell index per particle, per-cell counts,
                        prefix sum of the counts, out-of-place move into a
                        secondary array, interactions with the same and the
                        neighbouring cells, position update.
  PAPER.md:88-93  (§3)  inputs (positions, counts, start indices, values, SoA)
                        and outputs (forces, potential); cell width >= r_c.
  PAPER.md:236    (§5.1) each cell is used by 3^3 cells (27-neighbourhood).
  PAPER.md:839-864 (Appendix, Listing 1) the in-SM swap-free prefix sum.

Readings where the paper is silent are the DESIGN.md "Readings" table (Q-numbers
from SURVEY.md §8(c)); each is cited where it is used.
"""
from __future__ import annotations

import numpy as np

KERNEL_GAUSSIAN = 0
KERNEL_INDICATOR = 1
KERNEL_CANDIDATE = 2
KERNEL_LJ = 3
KERNEL_LOWFLOP = 4
KERNEL_HIGHFLOP = 5

# The kernel-cost sweep's fake kernels (Fig. "diffflops" caption; reading R22):
#   LOWFLOP  "a fake kernel that costs 5 FLOP per interaction (by summing the positions)":
#            c_ij = (x_j + y_j + z_j, x_j, y_j, z_j) for r_ij < r_c;
#   HIGHFLOP "the Lennard-Jones kernel with 150 added FLOP": the LJ potential term
#            u = (d~/r)^12 - (d~/r)^6 is run through HF_STEPS fused multiply-adds t <- t a + b
#            (2 FLOP each) before c_ij[0] = q_j 4 E0 t; the force is the LJ force.
HF_STEPS = 75
HF_A = 1.0 - 2.0 ** -7
HF_B = 2.0 ** -10


def highflop_chain(u):
    """The 150 added FLOP, step by step (reading R22)."""
    t = np.asarray(u, np.float64)
    for _ in range(HF_STEPS):
        t = t * HF_A + HF_B
    return t


def lj_params(grid):
    """(r, eps, E0) of the Lennard-Jones kernel, rounded to fp32 like every GPU input."""
    return (float(np.float32(grid.lj_ref)), float(np.float32(grid.lj_soft)), float(np.float32(grid.lj_e0)))


def lj_terms(r2, r, eps, e0):
    """Eq. (1) (§7.1) as printed, with the softening of PAPER.md:582 (reading
    R19): d~ = sqrt(d^2 + eps^2), u = d~ / r, K = 4 E0 (u^12 - u^6).  Returns K and
    G = -(dK/dd~) / d~ = -(4 E0 / r^2) (12 u^10 - 6 u^4), so that the force on i from j is
    q_i q_j G (x_i - x_j) = -grad_i (q_i q_j K)."""
    s = (r2 + eps * eps) / (r * r)  # u^2
    K = 4.0 * e0 * (s ** 6 - s ** 3)
    G = -(4.0 * e0 / (r * r)) * (12.0 * s ** 5 - 6.0 * s ** 2)
    return K, G


def lj_term_magnitudes(r2, r, eps, e0):
    """|contribution| scale of Eq. (1) per term (reading R20: the potential is
    the sum of the repulsive u^12 and the attractive u^6 term, each a contribution of its own):
    |K|_terms = 4 E0 (u^12 + u^6) and |G|_terms = (4 E0 / r^2) (12 u^10 + 6 u^4).  They bound the
    tolerance (C10) of the Lennard-Jones kernel, whose force term vanishes where 12 u^10 = 6 u^4
    while its two parts do not."""
    s = (r2 + eps * eps) / (r * r)
    return 4.0 * e0 * (s ** 6 + s ** 3), (4.0 * e0 / (r * r)) * (12.0 * s ** 5 + 6.0 * s ** 2)

# Ambiguity band for the cutoff decision (reading R15): pairs with
# |r^2 - r_c^2| <= BAND_REL * r_c^2 may be included or excluded by an fp32 implementation;
# their |contribution| is added to A_i.  An fp32 r^2 from rounded differences is within
# ~2^-21.7 r^2 of the exact value (tests/test_oracle.py::test_band_covers_fp32_r2 measures it).
BAND_REL = 2.0 ** -20


def band_rel(grid) -> float:
    return BAND_REL


# ------------------------------------------------------------------------------------
# a1: cell index (§2 "compute its cell index using its physical
# position").  Contract C3: c = clamp(floor(fl32(fl32(x - o) * inv_w)), 0, N-1)
# with inv_w = fl32(1 / w) and every fl32 operation rounded on its own (no FMA).
# numpy float32 arithmetic rounds per operation, which is exactly that contract.
# ------------------------------------------------------------------------------------

def inv_width(grid) -> np.float32:
    return np.float32(1.0) / np.float32(grid.w)


def cell_coords(x, y, z, grid):
    inv_w = inv_width(grid)
    out = []
    for a, o, nd in zip((x, y, z), grid.origin, grid.dims):
        a = np.asarray(a, dtype=np.float32)
        t = (a - np.float32(o)).astype(np.float32)
        t = (t * inv_w).astype(np.float32)
        c = np.floor(t.astype(np.float64)).astype(np.int64)
        c = np.clip(c, 0, int(nd) - 1)
        out.append(c)
    return tuple(out)


def linearize(cx, cy, cz, dims):
    """X-fastest linearisation (§5.1 'due to linearization'; reading Q3)."""
    nx, ny, _ = dims
    return cx + nx * (cy + ny * cz)


def cell_index(x, y, z, grid) -> np.ndarray:
    cx, cy, cz = cell_coords(x, y, z, grid)
    return linearize(cx, cy, cz, grid.dims).astype(np.int64)


# ------------------------------------------------------------------------------------
# a2-a3: counts, prefix array, M_C (PAPER.md:62-63 §2; :89 §3 "starting index of each
# cell in the sorted array"; :242 §5.1 "we retain the maximum number of particles in a
# cell when computing the prefix sum, denoted as M_C").  Layout: offsets[0] = 0,
# offsets[c+1] = offsets[c] + counts[c], offsets[Nc] = N (exclusive scan + total).
# ------------------------------------------------------------------------------------

def counts_of(cells: np.ndarray, ncells: int) -> np.ndarray:
    return np.bincount(np.asarray(cells, dtype=np.int64), minlength=ncells).astype(np.int64)


def prefix(counts: np.ndarray) -> np.ndarray:
    out = np.zeros(len(counts) + 1, dtype=np.int64)
    np.cumsum(counts, out=out[1:])
    return out


def sequential_prefix(counts) -> list:
    """Plain running sum, the definition the scan is pinned to."""
    out = [0]
    for c in counts:
        out.append(out[-1] + int(c))
    return out


def max_per_cell(counts: np.ndarray) -> int:
    return int(counts.max()) if len(counts) else 0


def members(cells: np.ndarray, ncells: int) -> dict:
    """C5: cell -> set of particle indices (order inside a cell is free: the paper's
    scatter takes slots with atomics)."""
    d = {}
    for i, c in enumerate(np.asarray(cells).tolist()):
        d.setdefault(c, set()).add(i)
    return d


# ------------------------------------------------------------------------------------
# C6: the 27-neighbourhood, clamped at the open box boundary (§5.1;
# boundaries are open: reading Q2, pinned by Table 1's interactions-per-particle
# column, tests/test_oracle.py::test_table1_ipp).
# ------------------------------------------------------------------------------------

def neighbour_coords(cx, cy, cz, dims):
    nx, ny, nz = dims
    out = []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                a, b, c = cx + dx, cy + dy, cz + dz
                if 0 <= a < nx and 0 <= b < ny and 0 <= c < nz:
                    out.append((a, b, c))
    return out


def candidate_mask(cc_i, cc_j):
    """Candidate pair <=> Chebyshev distance between the two cells <= 1."""
    return np.max(np.abs(cc_i - cc_j), axis=-1) <= 1


# ------------------------------------------------------------------------------------
# a6: interactions, O(N^2) brute force (§2).  For every i and every
# j != i (identity, Alg. 1 :127 "part_source != part_target"; reading Q7) with
# r_ij < r_c (strict, reading Q5):
#   Gaussian  (PAPER.md:52 names the Gaussian; definition = reading Q8 / C8):
#     K(r) = exp(-r^2 / (2 sigma^2));  c_ij = (q_j K, q_i q_j K (x_i - x_j)/sigma^2, ...)
#     phi_i = sum_j c_ij[0],  F_i = sum_j c_ij[1:4]   (F_i = -grad_i sum_j q_i q_j K)
#   LJ:        c_ij = (q_j K, q_i q_j G (x_i - x_j)), K, G of lj_terms (Eq. (1), reading R19)
#   INDICATOR: c_ij = (q_j, 0, 0, 0) inside the cutoff (test kernel)
#   CANDIDATE: c_ij = (q_j, 0, 0, 0) for every candidate pair, no cutoff (test kernel)
# Returned alongside: S_i = sum |c_ij| over included pairs (per component; for LJ the
# per-term magnitudes of lj_term_magnitudes, reading R20),
# A_i = sum |c_ij| over ambiguous pairs (|r^2 - r_c^2| <= band * r_c^2), the candidate
# count C_i and the cutoff-pair count P_i.  Accumulation in fp64 (C9).
# ------------------------------------------------------------------------------------

def brute_force(x, y, z, q, grid, kernel=KERNEL_GAUSSIAN, band=None, chunk=512):
    n = len(x)
    X = np.stack([np.asarray(x, np.float64), np.asarray(y, np.float64), np.asarray(z, np.float64)], axis=1)
    Q = np.asarray(q, np.float64)
    cc = np.stack(cell_coords(x, y, z, grid), axis=1)
    rc = float(np.float32(grid.r_c))
    rc2 = rc * rc
    sig = float(np.float32(grid.sig))
    inv2s2 = 1.0 / (2.0 * sig * sig)
    if band is None:
        band = band_rel(grid)
    out = np.zeros((n, 4))
    S = np.zeros((n, 4))
    A = np.zeros((n, 4))
    C = np.zeros(n, dtype=np.int64)
    P = np.zeros(n, dtype=np.int64)
    idx = np.arange(n)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        d = X[s:e, None, :] - X[None, :, :]               # x_i - x_j
        r2 = np.einsum("ijk,ijk->ij", d, d)
        notself = idx[s:e, None] != idx[None, :]
        cand = candidate_mask(cc[s:e, None, :], cc[None, :, :]) & notself
        inside = (r2 < rc2) & notself
        # with w >= r_c every pair inside the cutoff is a candidate
        assert not np.any(inside & ~cand), "pair inside r_c outside the 27-neighbourhood"
        amb = (np.abs(r2 - rc2) <= band * rc2) & cand
        if kernel == KERNEL_GAUSSIAN:
            K = np.exp(-r2 * inv2s2)
            c0 = Q[None, :] * K
            cf = (Q[s:e, None] * Q[None, :] * K / (sig * sig))[:, :, None] * d
            comps = np.concatenate([c0[:, :, None], cf], axis=2)
            incl = inside
        elif kernel == KERNEL_LJ:
            K, G = lj_terms(r2, *lj_params(grid))
            c0 = Q[None, :] * K
            cf = (Q[s:e, None] * Q[None, :] * G)[:, :, None] * d
            comps = np.concatenate([c0[:, :, None], cf], axis=2)
            Km, Gm = lj_term_magnitudes(r2, *lj_params(grid))  # reading R20: per-term |c_ij|
            m0 = np.abs(Q[None, :]) * Km
            mf = np.abs(Q[s:e, None] * Q[None, :] * Gm)[:, :, None] * np.abs(d)
            mags = np.concatenate([m0[:, :, None], mf], axis=2)
            incl = inside
        elif kernel == KERNEL_HIGHFLOP:
            r_, eps_, e0_ = lj_params(grid)
            K, G = lj_terms(r2, r_, eps_, e0_)
            u = K / (4.0 * e0_)                                 # (d~/r)^12 - (d~/r)^6
            c0 = Q[None, :] * 4.0 * e0_ * highflop_chain(u)
            cf = (Q[s:e, None] * Q[None, :] * G)[:, :, None] * d
            comps = np.concatenate([c0[:, :, None], cf], axis=2)
            Km, Gm = lj_term_magnitudes(r2, r_, eps_, e0_)
            # |terms| of the chain: A |u|_terms + sum_k b a^k = A |u|_terms + B (A = a^75)
            A_ = HF_A ** HF_STEPS
            m0 = np.abs(Q[None, :]) * 4.0 * e0_ * (A_ * Km / (4.0 * e0_) + HF_B * (1.0 - A_) / (1.0 - HF_A))
            mf = np.abs(Q[s:e, None] * Q[None, :] * Gm)[:, :, None] * np.abs(d)
            mags = np.concatenate([m0[:, :, None], mf], axis=2)
            incl = inside
        elif kernel == KERNEL_LOWFLOP:
            comps = np.zeros(r2.shape + (4,))
            Xj = X[None, :, :] * np.ones((e - s, 1, 1))
            comps[:, :, 0] = Xj.sum(axis=2)
            comps[:, :, 1:] = Xj
            incl = inside
        elif kernel == KERNEL_INDICATOR:
            comps = np.zeros(r2.shape + (4,))
            comps[:, :, 0] = Q[None, :]
            incl = inside
        elif kernel == KERNEL_CANDIDATE:
            comps = np.zeros(r2.shape + (4,))
            comps[:, :, 0] = Q[None, :]
            incl = cand
            amb = np.zeros_like(amb)
        else:
            raise ValueError(kernel)
        if kernel not in (KERNEL_LJ, KERNEL_HIGHFLOP):
            mags = np.abs(comps)
        if kernel == KERNEL_LOWFLOP:  # per component term: |x_j| + |y_j| + |z_j| for phi
            mags = np.abs(comps)
            mags[:, :, 0] = np.abs(Xj).sum(axis=2)
        out[s:e] = np.einsum("ij,ijk->ik", incl.astype(np.float64), comps)
        S[s:e] = np.einsum("ij,ijk->ik", incl.astype(np.float64), mags)
        A[s:e] = np.einsum("ij,ijk->ik", amb.astype(np.float64), mags)
        C[s:e] = cand.sum(axis=1)
        P[s:e] = inside.sum(axis=1)
    return dict(out=out, S=S, A=A, C=C, P=P)


def check_interactions(gpu, ref, rel=1e-4):
    """C10 acceptance: |gpu - oracle| <= rel * S_i + A_i per particle and component;
    exact 0 where S_i = A_i = 0.  gpu: (n, 4) array (phi, fx, fy, fz).
    Returns (ok, worst_ratio, index_of_worst)."""
    gpu = np.asarray(gpu, np.float64)
    err = np.abs(gpu - ref["out"])
    bound = rel * ref["S"] + ref["A"]
    zero = (ref["S"] == 0) & (ref["A"] == 0)
    bad_zero = zero & (gpu != 0)
    with np.errstate(divide="ignore", invalid="ignore"):
        ratio = np.where(bound > 0, err / np.where(bound > 0, bound, 1), np.where(err > 0, np.inf, 0))
    worst = float(np.max(ratio)) if ratio.size else 0.0
    ok = (not np.any(bad_zero)) and worst <= 1.0
    return ok, worst, np.unravel_index(int(np.argmax(ratio)), ratio.shape) if ratio.size else None


# ------------------------------------------------------------------------------------
# a7: position update (§2 "their positions are updated"; the scheme is
# unstated -> reading Q11 / C11): x' = x + dt F, then reflect at the walls
# (x < o -> 2o - x; x >= o + L -> 2(o + L) - x), then clamp into [o, o + L).
# Evaluated in fp64 from fp32 inputs; compared with tolerance dt*(rel*S_F + A_F) + ulp.
# ------------------------------------------------------------------------------------

def integrate(x, f, dt, lo, hi):
    x = np.asarray(x, np.float64) + dt * np.asarray(f, np.float64)
    x = np.where(x < lo, 2 * lo - x, x)
    x = np.where(x >= hi, 2 * hi - x, x)
    below = float(np.nextafter(np.float32(hi), np.float32(lo)))
    return np.clip(x, lo, below)


# ------------------------------------------------------------------------------------
# The paper's in-SM prefix sum, sequentialised (Appendix Listing 1, PAPER.md:839-864;
# §6 Alg. 6 :502-531).  `reset` selects the downward-pass start: "listing" =
# js = max(4, js/2), "alg6" = js = max(4, js/4).
# Returns the inclusive prefix sum in place and the intermediate states of each pass.
# Used only as a pinned worked example; the CUDA path scans with
# warp shuffles and decoupled look-back instead.
# ------------------------------------------------------------------------------------

def paper_inplace_scan(values, reset="listing"):
    a = list(values)
    n = len(a)
    states = []
    js = 2
    while js <= n:
        jsd2 = js // 2
        for idn in range(js - 1, n, js):
            a[idn] = a[idn] + a[idn - jsd2]
        states.append(list(a))
        js *= 2
    js = max(4, js // 2) if reset == "listing" else max(4, js // 4)
    while js > 1:
        jsd2 = js // 2
        for idn in range(js + jsd2 - 1, n, js):
            a[idn] = a[idn] + a[idn - jsd2]
        states.append(list(a))
        js = jsd2
    return a, states


# ------------------------------------------------------------------------------------
# Full-load local offsets, "gap" reading of PAPER.md:321-327 (§5.1, Fig. local offset;
# reading Q19 / C7).  For a sub-box X-range [x0, x1] and its pencils p = (y, z) in
# Z-outer / Y-inner order:  n_p = off[lin(x1,p)+1] - off[lin(x0,p)];
# g_0 = off[lin(x0,p_0)], g_p = off[lin(x0,p)] - off[lin(x1,p-1)+1];
# E_p = sum_{p'<=p} g_p';  local(c) = off[c] - E_p.
# ------------------------------------------------------------------------------------

def subbox_local_offsets(offsets, dims, x0, x1, y0, y1, z0, z1):
    nx, ny, _ = dims
    lin = lambda a, b, c: a + nx * (b + ny * c)
    pencils = [(yy, zz) for zz in range(z0, z1 + 1) for yy in range(y0, y1 + 1)]
    local = {}
    E = 0
    prev_end = None
    for k, (yy, zz) in enumerate(pencils):
        start = int(offsets[lin(x0, yy, zz)])
        g = start if k == 0 else start - prev_end
        E += g
        for xx in range(x0, x1 + 1):
            c = lin(xx, yy, zz)
            local[c] = int(offsets[c]) - E
        prev_end = int(offsets[lin(x1, yy, zz) + 1])
    return local
