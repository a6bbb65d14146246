"""a5-a6 parity through the C ABI: every strategy and kernel against the fp64 oracle.

Tolerance (north star / C10): |gpu - oracle| <= 1e-4 * sum_j |c_ij| + A_i per particle and
component, exact 0 where nothing contributes; INDICATOR / CANDIDATE counts (q = 1) exact."""
import numpy as np
import pytest
import torch

import synth
from oracle import celllist
from oracle import reference as ref
from tests._util import assert_parity, ctx_for, gpu_interact, oracle_interact, to_dev

pytestmark = pytest.mark.gpu
ALGOS = ["global", "xpencil", "fullload", "xpreg", "half"]
# Every strategy computes r^2 from differences of the raw fp32 positions: for dyadic inputs
# every step is exact, so pairs at exactly r = r_c are excluded exactly (band 0) by all of them.


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("kernel", ["gaussian", "indicator", "candidate", "lj", "lowflop", "highflop"])
def test_c0_full(algo, kernel):
    """configs[0]: 4096 uniform particles, 16^3 cells, every particle vs the oracle."""
    c = synth.make_config("c0")
    got, ctx = gpu_interact(c, algo, kernel)
    want = oracle_interact(c, kernel)
    assert_parity(got, want, label=f"c0 {algo} {kernel}")
    if kernel in ("indicator", "candidate"):
        assert np.all(got[:, 1:] == 0)
    st = ctx.stats()
    assert st["candidates"] == int(want["C"].sum())


@pytest.mark.parametrize("algo", ALGOS)
def test_counts_exact_q1(algo):
    c = synth.make_config("c0", qkind="ones")
    got, _ = gpu_interact(c, algo, "indicator")
    want = oracle_interact(c, "indicator")
    assert np.array_equal(got[:, 0], want["P"].astype(np.float64))
    got, _ = gpu_interact(c, algo, "candidate")
    want = oracle_interact(c, "candidate")
    assert np.array_equal(got[:, 0], want["C"].astype(np.float64))


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("variant", ["A", "B"])
def test_hand2x3_exact(algo, variant):
    """C12: dyadic coordinates; variant B has pairs at exactly r = r_c that must be excluded."""
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hand2x3.json")))
    band = 0.0   # variant B has pairs at exactly r_c: excluded exactly
    c = synth.hand_2x3(variant)
    c.q = np.ones(9, np.float32)
    got, _ = gpu_interact(c, algo, "candidate")
    assert got[:, 0].tolist() == g["candidate_q1"]
    got, _ = gpu_interact(c, algo, "indicator")
    assert got[:, 0].tolist() == g["indicator_q1"]
    assert_parity(got, oracle_interact(c, "indicator", band=band), label="hand indicator")
    c = synth.hand_2x3(variant)
    got, _ = gpu_interact(c, algo, "indicator")
    assert got[:, 0].tolist() == g["indicator_qj"]
    want = oracle_interact(c, "gaussian", band=band)
    got, _ = gpu_interact(c, algo, "gaussian")
    assert_parity(got, want, label="hand gaussian")


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("d", [4, 8])
def test_lattice_exact_boundary(algo, d):
    """C14: dyadic lattice with pairs at exactly r = r_c (band 0): interior phi/q closed form."""
    c = synth.lattice(d)
    band = 0.0
    got, _ = gpu_interact(c, algo, "indicator")
    want = oracle_interact(c, "indicator", band=band)
    assert np.array_equal(got[:, 0], want["P"].astype(np.float64))
    assert_parity(got, want, label=f"lattice{d} {algo} indicator")
    got, _ = gpu_interact(c, algo, "gaussian")
    want = oracle_interact(c, "gaussian", band=band)
    assert_parity(got, want, label=f"lattice{d} {algo}")


@pytest.mark.parametrize("algo", ALGOS)
def test_degenerate(algo):
    grid = synth.Grid(dims=(4, 4, 4), w=0.25)
    # one particle: exactly zero
    c = synth.Cloud(grid, np.array([0.3], np.float32), np.array([0.6], np.float32), np.array([0.9], np.float32),
                    np.array([1.5], np.float32))
    got, _ = gpu_interact(c, algo)
    assert np.all(got == 0)
    # two particles in neighbouring cells, closed form
    c = synth.Cloud(grid, np.array([0.30, 0.40], np.float32), np.array([0.30, 0.35], np.float32),
                    np.array([0.30, 0.28], np.float32), np.array([1.25, 0.75], np.float32))
    got, _ = gpu_interact(c, algo)
    assert_parity(got, oracle_interact(c), label="two")
    # coincident distinct particles do interact (identity exclusion, K(0) = 1, F = 0)
    c = synth.Cloud(grid, np.array([0.3, 0.3], np.float32), np.array([0.3, 0.3], np.float32),
                    np.array([0.3, 0.3], np.float32), np.array([2.0, 3.0], np.float32))
    got, _ = gpu_interact(c, algo)
    assert got[0, 0] == pytest.approx(3.0, rel=1e-6) and got[1, 0] == pytest.approx(2.0, rel=1e-6)
    assert np.all(got[:, 1:] == 0)
    # empty
    c = synth.Cloud(grid, *(np.zeros(0, np.float32) for _ in range(4)))
    ctx = ctx_for(c, capacity=16)
    ctx.bin(*to_dev(c))
    ctx.interact(algo)
    torch.cuda.synchronize()


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("ppc", [1, 4, 8, 20, 64])
def test_density_sweep(algo, ppc):
    """BASELINE configs[2] shape (particles-per-cell sweep) at oracle-friendly sizes."""
    c = synth.scaled_uniform(ppc, (12, 10, 9), seed=240616093 + ppc)
    got, _ = gpu_interact(c, algo)
    assert_parity(got, oracle_interact(c), label=f"ppc{ppc} {algo}")


@pytest.mark.parametrize("algo", ALGOS)
def test_signed_charges(algo):
    c = synth.make_config("c0", qkind="signed")
    got, _ = gpu_interact(c, algo)
    assert_parity(got, oracle_interact(c), label="signed")


@pytest.mark.parametrize("algo", ALGOS)
def test_clustered_small(algo):
    """configs[3] shape at 2^17 particles on 32^3: dense blobs exercise the staging overflow path."""
    c = synth.clustered(1 << 17, synth.Grid(dims=(32, 32, 32), w=1 / 32), seed=240616094)
    got, ctx = gpu_interact(c, algo)
    sample = np.random.default_rng(1).choice(c.n, 20000, replace=False)
    want = oracle_interact(c, targets=sample)
    assert_parity(got[sample], want, label=f"clustered {algo}")


@pytest.mark.parametrize("algo", ALGOS)
def test_xpencil_tuning_shapes(algo):
    """Staged kernel with tiny capacity (forces several rounds and the fallback) and odd lengths."""
    c = synth.scaled_uniform(8, (20, 6, 5), seed=3)
    want = oracle_interact(c)
    for tune in (dict(xpencil_len=1), dict(xpencil_len=7, xpencil_cap=300), dict(xpencil_len=64),
                 dict(xpencil_len=16, xpencil_cap=64), dict(threads=256, xpencil_len=5), dict(threads=32),
                 dict(xpencil_cap=16), dict(xpencil_slots=3), dict(xpencil_slots=4, xpencil_len=16),
                 dict(xpencil_slots=4, threads=256), dict(xpencil_slots=5),
                 dict(xpencil_targets=2), dict(xpencil_targets=2, xpencil_len=7, xpencil_cap=300),
                 dict(xpencil_targets=2, xpencil_cap=64), dict(xpencil_targets=2, threads=288),
                 dict(xpencil_targets=3), dict(xpencil_targets=3, xpencil_len=7, xpencil_cap=300),
                 dict(xpencil_targets=3, xpencil_cap=64), dict(xpencil_targets=3, threads=288)):
        got, ctx = gpu_interact(c, algo, tuning=tune)
        assert_parity(got, want, label=f"{algo} {tune}")
        if algo == "xpencil" and tune.get("xpencil_cap") in (16, 64):
            assert ctx.stats()["fallback_cells"] > 0  # merged cells over the cap take the global path


def test_fullload_tuning_shapes():
    """Full-load sub-box dims (incl. 1x1x1 = 27 staged cells) and a capacity too
    small for the sub-box (global-memory fallback of the whole block)."""
    c = synth.scaled_uniform(8, (20, 6, 5), seed=4)
    want = oracle_interact(c)
    for tune in (dict(fullload_box=(1, 1, 1)), dict(fullload_box=(3, 2, 5)), dict(fullload_box=(20, 6, 5)),
                 dict(fullload_box=(8, 4, 4), fullload_cap=64), dict(fullload_box=(4, 4, 4), threads=128),
                 dict(threads=512)):
        got, ctx = gpu_interact(c, "fullload", tuning=tune)
        assert_parity(got, want, label=f"fullload {tune}")
    assert ctx.stats()["candidates"] == int(want["C"].sum())


@pytest.mark.parametrize("algo", ALGOS)
def test_c1_sampled(algo):
    """configs[1] (2^21, 64^3, 8/cell) in the bench's launch configuration, sampled targets."""
    c = synth.make_config("c1")
    got, ctx = gpu_interact(c, algo)
    sample = np.random.default_rng(2).choice(c.n, 30000, replace=False)
    want = oracle_interact(c, targets=sample)
    assert_parity(got[sample], want, label=f"c1 {algo}")
    st = ctx.stats()
    assert st["fallback_cells"] == 0
    # property at full size: sum of forces ~ 0 (antisymmetry), relative to sum |F|
    F = got[:, 1:]
    assert np.all(np.abs(F.sum(0)) <= 1e-4 * np.abs(F).sum(0))


@pytest.mark.parametrize("xs", [1, 2, 4, 8, 16])
@pytest.mark.parametrize("kernel", ["gaussian", "indicator", "candidate", "lj"])
def test_x_subcells(xs, kernel):
    """Binning order with X sub-cells (R18): per-cell counts/offsets unchanged (bit-exact), and the
    X-pencil's pruning of sub-cells farther than r_c along X changes no result."""
    c = synth.scaled_uniform(8, (20, 6, 5), seed=7)
    want = oracle_interact(c, kernel)
    ctx = ctx_for(c, kernel, x_subcells=xs)
    for algo in ALGOS:
        got, _ = gpu_interact(c, algo, kernel, ctx=ctx)
        assert_parity(got, want, label=f"x_subcells={xs} {kernel} {algo}")
    ctx.set_tuning(xpencil_targets=2)  # union windows of two consecutive targets per lane
    got, _ = gpu_interact(c, "xpencil", kernel, ctx=ctx)
    assert_parity(got, want, label=f"x_subcells={xs} {kernel} xpencil two targets per lane")
    ctx.set_tuning()
    counts, offsets = (t.cpu().numpy() for t in ctx.get_offsets())
    wc, wo, _ = celllist.binning(celllist.cells(c.x, c.y, c.z, c.grid), c.grid.ncells)
    assert np.array_equal(counts, wc) and np.array_equal(offsets, wo)
    assert ctx.stats()["max_per_cell"] == int(wc.max())


@pytest.mark.parametrize("nx", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("kernel", ["gaussian", "indicator", "lj"])
def test_narrow_x(nx, kernel):
    """Grids of 1-5 cells along X: below 4 cells the X-pencil masks the out-of-run halves of a
    run's end pairs (their partner records can then be within r_c across a row end)."""
    c = synth.scaled_uniform(8, (nx, 7, 6), seed=11 + nx)
    want = oracle_interact(c, kernel)
    for algo in ALGOS:
        got, _ = gpu_interact(c, algo, kernel)
        assert_parity(got, want, label=f"nx={nx} {kernel} {algo}")


@pytest.mark.parametrize("algo", ALGOS)
def test_lj_softening_coincident_and_params(algo):
    """Eq. (1) with softening (R19): coincident distinct particles interact through K(eps) with no
    force; an isolated particle is exactly 0; non-default r, eps, E0 reach every strategy."""
    grid = synth.Grid(dims=(4, 4, 4), w=0.25, lj_r=0.25, lj_eps=0.125, lj_e0=2.0)
    c = synth.Cloud(grid, np.array([0.3, 0.3, 0.9], np.float32), np.array([0.3, 0.3, 0.9], np.float32),
                    np.array([0.3, 0.3, 0.9], np.float32), np.array([2.0, 3.0, 1.0], np.float32))
    got, _ = gpu_interact(c, algo, "lj")
    K = 4 * 2.0 * (0.5 ** 12 - 0.5 ** 6)
    assert got[0, 0] == pytest.approx(3.0 * K, rel=1e-6) and got[1, 0] == pytest.approx(2.0 * K, rel=1e-6)
    assert np.all(got[:2, 1:] == 0) and np.all(got[2] == 0)
    c2 = synth.scaled_uniform(8, (10, 8, 6), seed=21)
    c2.grid = synth.Grid(dims=c2.grid.dims, w=c2.grid.w, lj_r=0.8 * c2.grid.w, lj_eps=0.03 * c2.grid.w, lj_e0=0.7)
    got, _ = gpu_interact(c2, algo, "lj")
    assert_parity(got, oracle_interact(c2, "lj"), label=f"lj params {algo}")


@pytest.mark.parametrize("algo", ALGOS)
def test_run_host_paths(algo):
    """End-to-end calls on pinned host buffers: the synchronous pi_run_host and the pipelined
    pi_run_host_submit/_wait (two runs in flight on alternating I/O sets, a third submit waits
    for the oldest) give the oracle's values for each of several different inputs."""
    clouds = [synth.scaled_uniform(8, (12, 10, 9), seed=s) for s in (21, 22, 23, 24, 25)]
    wants = [oracle_interact(c) for c in clouds]
    cap = max(c.n for c in clouds)
    ctx = ctx_for(clouds[0], capacity=cap)
    pin = lambda a: torch.from_numpy(a).pin_memory()
    hin = [[pin(a) for a in (c.x, c.y, c.z, c.q)] for c in clouds]
    hout = [[torch.full((c.n,), float("nan")).pin_memory() for _ in range(4)] for c in clouds]
    ctx.run_host(algo, *hin[0], *hout[0])
    assert_parity(torch.stack(hout[0], 1).numpy(), wants[0], label=f"run_host {algo}")
    for o in hout[0]:
        o.fill_(float("nan"))
    for k in range(len(clouds)):
        ctx.run_host_submit(algo, *hin[k], *hout[k])
    ctx.run_host_wait()
    for k in range(len(clouds)):
        assert_parity(torch.stack(hout[k], 1).numpy(), wants[k], label=f"run_host_submit {algo} run {k}")


# Lennard-Jones included: its tolerance scale is per Eq. (1) term (reading R20), so a pair near
# the zero of the LJ force (12 u^10 = 6 u^4), where the fp32 term cancels, is covered.
@pytest.mark.parametrize("kernel", ["gaussian", "indicator", "candidate", "lj"])
@pytest.mark.parametrize("xcap", [16, 200])
def test_dense_cells_par_cell_sm(kernel, xcap):
    """Cells whose window alone does not fit an X-pencil slot are listed and computed by the
    Par-Cell-SM pass: a staging capacity of 16 lists every cell, 200 some.
    Clustered cloud (configs[3] recipe, small): parity, exact integer counts, exact candidates."""
    qk = "ones" if kernel in ("indicator", "candidate") else "pos"
    c = synth.clustered(1 << 14, synth.Grid(dims=(16, 16, 16), w=1 / 16), seed=240616094, qkind=qk)
    want = oracle_interact(c, kernel)
    got, ctx = gpu_interact(c, "xpencil", kernel, tuning=dict(xpencil_cap=xcap))
    assert_parity(got, want, label=f"dense {kernel} cap {xcap}")
    if qk == "ones":  # integer outputs: exact
        assert np.array_equal(got[:, 0], want["P" if kernel == "indicator" else "C"].astype(np.float64))
    st = ctx.stats()
    assert st["fallback_cells"] > 0
    assert st["candidates"] == int(want["C"].sum())


@pytest.mark.parametrize("name", ["c3", "c2_ppc1", "c2_ppc64"])
def test_full_size_sampled(name):
    """BASELINE configs at full size (2^24 particles) in the bench's launch configuration,
    sampled targets against the oracle: configs[3] clustered (M_C ~ 370: the X-pencil lists its
    densest cells for the Par-Cell-SM pass) and the two ends of the configs[2] ppc sweep (1 and
    64 per cell).  Candidates are checked against the oracle's count on the sample's cells'
    closed form at full size, from the ORACLE's own binning: sum over cells of n_c (sum of the 27
    neighbours' counts) - N."""
    c = synth.make_config(name)
    ctx = ctx_for(c)
    got, ctx = gpu_interact(c, "xpencil", ctx=ctx)
    sample = np.random.default_rng(5).choice(c.n, 4000, replace=False)
    want = oracle_interact(c, targets=sample)
    assert_parity(got[sample], want, label=f"{name} xpencil")
    assert ctx.stats()["candidates"] == oracle_candidates(c)
    if name == "c3":
        assert ctx.stats()["fallback_cells"] > 0


def oracle_candidates(c):
    """C = sum_c n_c (sum of the 27 clamped neighbours' counts) - N from the oracle's binning."""
    counts = ref.counts_of(celllist.cells(c.x, c.y, c.z, c.grid), c.grid.ncells)
    nx, ny, nz = c.grid.dims
    n3 = counts.reshape(nz, ny, nx)
    pad = np.pad(n3, 1)
    nb = sum(pad[1 + dz:1 + dz + nz, 1 + dy:1 + dy + ny, 1 + dx:1 + dx + nx]
             for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1))
    return int((n3 * nb).sum() - c.n)


@pytest.mark.parametrize("algo", ["global", "fullload", "xpreg", "half"])
def test_full_size_other_strategies(algo):
    """The global baseline and the full load at full size: configs[2] ppc 8 (2^24 on 128^3),
    sampled targets against the oracle, candidates against the oracle's closed form."""
    c = synth.make_config("c2_ppc8")
    got, ctx = gpu_interact(c, algo)
    sample = np.random.default_rng(6).choice(c.n, 4000, replace=False)
    assert_parity(got[sample], oracle_interact(c, targets=sample), label=f"c2_ppc8 {algo}")
    assert ctx.stats()["candidates"] == oracle_candidates(c)


def test_c4_full_size_sampled():
    """configs[4] on one GPU (2^27 uniform, 256^3 cells: the bench's workload) with the bench's
    strategy: sampled targets against the oracle, candidates against its closed form."""
    c = synth.make_config("c4")
    got, ctx = gpu_interact(c, "xpencil")
    sample = np.random.default_rng(7).choice(c.n, 3000, replace=False)
    assert_parity(got[sample], oracle_interact(c, targets=sample), label="c4 xpencil")
    assert ctx.stats()["candidates"] == oracle_candidates(c)


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("kernel", ["lowflop", "highflop"])
@pytest.mark.parametrize("ppc", [2, 20])
def test_cost_sweep_kernels(algo, kernel, ppc):
    """The kernel-cost sweep's fake kernels (reading R22) at two densities, and
    an isolated particle exactly 0 (the self pair removed exactly, positions included)."""
    c = synth.scaled_uniform(ppc, (12, 10, 9), seed=240616097 + ppc)
    got, _ = gpu_interact(c, algo, kernel)
    assert_parity(got, oracle_interact(c, kernel), label=f"{kernel} ppc{ppc} {algo}")
    grid = synth.Grid(dims=(4, 4, 4), w=0.25)
    one = synth.Cloud(grid, np.array([0.3], np.float32), np.array([0.6], np.float32), np.array([0.9], np.float32),
                      np.array([1.5], np.float32))
    got, _ = gpu_interact(one, algo, kernel)
    assert np.all(got == 0)


@pytest.mark.parametrize("name", ["c0", "c1"])
def test_count_pairs(name):
    """pi_count_pairs (P) equals the oracle's sum of P_i, after pi_bin (records) and
    after a pi_step that left only the source-pair array of the re-binned state.  Exact up to the
    pairs inside the fp32/fp64 ambiguity band (R15), counted by the oracle (q = 1: A_i[0])."""
    c = synth.make_config(name, qkind="ones")
    ctx = ctx_for(c)
    ctx.bin(*to_dev(c))
    want = oracle_interact(c, "indicator")
    P, amb = int(want["P"].sum()), int(want["A"][:, 0].sum())
    assert abs(ctx.count_pairs() - P) <= amb
    ctx.step("xpencil", 0.0)
    ctx.step("xpencil", 0.0)    # dt = 0: the re-binned state (pair array only) is the same cloud
    assert abs(ctx.count_pairs() - P) <= amb


def test_xpencil_fine_subcells_wide_grid():
    """x_subcells = 16 on a grid 256 cells wide at 1-2 particles per cell: the X-pencil's segment
    is sized from the shared-memory budget too (it used to need more than 227 KB for
    its tables alone and returned PI_EINAPPLICABLE)."""
    c = synth.scaled_uniform(1.5, (256, 8, 8), seed=240616099)
    want = oracle_interact(c)
    got, ctx = gpu_interact(c, "xpencil", ctx=ctx_for(c, x_subcells=16))
    assert_parity(got, want, label="sx16 wide")
    assert ctx.stats()["candidates"] == int(want["C"].sum())


def test_run_host_after_submits():
    """pi_run_host while pipelined runs are in flight drains them first (it shares
    their I/O set 0): every run's host output is the oracle's."""
    clouds = [synth.scaled_uniform(8, (12, 10, 9), seed=s) for s in (31, 32, 33)]
    wants = [oracle_interact(c) for c in clouds]
    ctx = ctx_for(clouds[0], capacity=max(c.n for c in clouds))
    pin = lambda a: torch.from_numpy(a).pin_memory()
    hin = [[pin(a) for a in (c.x, c.y, c.z, c.q)] for c in clouds]
    hout = [[torch.full((c.n,), float("nan")).pin_memory() for _ in range(4)] for c in clouds]
    ctx.run_host_submit("xpencil", *hin[0], *hout[0])
    ctx.run_host_submit("xpencil", *hin[1], *hout[1])
    ctx.run_host("xpencil", *hin[2], *hout[2])   # no wait in between
    ctx.run_host_wait()
    for k in range(3):
        assert_parity(torch.stack(hout[k], 1).numpy(), wants[k], label=f"run {k}")


@pytest.mark.parametrize("kernel", ["gaussian", "indicator", "candidate", "lj", "lowflop", "highflop"])
def test_xpencil_interleaved_layout(kernel):
    """The X-pencil's sub-cell-interleaved staging (tuning xpencil_layout = 1): configs[0] against
    the oracle for every kernel, a clustered cloud with dense cells, and exact integer counts."""
    c = synth.make_config("c0")
    got, ctx = gpu_interact(c, "xpencil", kernel, tuning=dict(xpencil_layout=1))
    want = oracle_interact(c, kernel)
    assert_parity(got, want, label=f"interleaved {kernel}")
    assert ctx.stats()["candidates"] == int(want["C"].sum())
    if kernel in ("indicator", "candidate"):
        c1 = synth.make_config("c0", qkind="ones")
        got, _ = gpu_interact(c1, "xpencil", kernel, tuning=dict(xpencil_layout=1))
        w = oracle_interact(c1, kernel)
        assert np.array_equal(got[:, 0], w["P" if kernel == "indicator" else "C"].astype(np.float64))
    cl = synth.clustered(1 << 14, synth.Grid(dims=(16, 16, 16), w=1 / 16), seed=240616094)
    got, ctx = gpu_interact(cl, "xpencil", kernel, tuning=dict(xpencil_layout=1, xpencil_cap=200))
    assert_parity(got, oracle_interact(cl, kernel), label=f"interleaved clustered {kernel}")


@pytest.mark.parametrize("seed", range(12))
def test_xpencil_tuning_fuzz(seed):
    """Random X-pencil launch shapes (segment length, slot capacity small enough to force rounds
    and listed dense cells, 2-4 slots, X sub-cells, grid shape, density, kernel) against the
    oracle: the producer / helper hand-over of offsets tables across rounds and slots, the
    Par-Cell-SM listing and the windows must give the same sums in every combination."""
    rng = np.random.default_rng(1000 + seed)
    dims = tuple(int(v) for v in rng.integers(4, 14, size=3))
    ppc = float(rng.choice([2, 5, 9, 16]))
    if seed % 3:
        c = synth.scaled_uniform(ppc, dims, seed=77 + seed)
    else:  # clustered blobs in the unit box: a cubic grid of width 1/d (non-dyadic for most d)
        d = dims[0]
        c = synth.clustered(int(ppc * d ** 3), synth.Grid(dims=(d, d, d), w=1 / d), seed=88 + seed)
    kernel = ["gaussian", "indicator", "candidate", "lj"][seed % 4]
    xs = int(rng.choice([1, 2, 4, 8]))
    tune = dict(xpencil_len=int(rng.integers(1, 20)), xpencil_cap=int(rng.choice([0, 48, 96, 300, 1000])),
                xpencil_slots=int(rng.integers(2, 5)))
    want = oracle_interact(c, kernel)
    ctx = ctx_for(c, kernel, x_subcells=xs)
    got, ctx = gpu_interact(c, "xpencil", kernel, tuning=tune, ctx=ctx)
    assert_parity(got, want, label=f"fuzz {seed} dims {dims} ppc {ppc} sx {xs} {kernel} {tune}")
    assert ctx.stats()["candidates"] == int(want["C"].sum())


def test_out_of_box_flag():
    """pi.h: a position outside [origin, origin + dims w] raises flag 1 (PI_EDEVICE at the next
    pi_get_stats); a particle exactly on the upper face is in the box (it clamps into the last
    cell) and raises nothing."""
    from paper_2406_16091_b200 import PiError
    c = synth.make_config("c0")
    c.x[:8] = 1.0  # the upper face x = 16 w: legal
    ctx = ctx_for(c)
    ctx.bin(*to_dev(c))
    ctx.interact("xpencil")
    ctx.stats()
    for bad in (1.0 + 1 / 64, -1e-3, float("nan")):
        c2 = synth.make_config("c0")
        c2.y[5] = np.float32(bad)
        ctx = ctx_for(c2)
        ctx.bin(*to_dev(c2))
        with pytest.raises(PiError, match="0x1"):
            ctx.stats()


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("algo", ["global", "fullload", "xpreg", "half"])
def test_strategy_fuzz(algo, seed):
    """Random grid shapes, densities, X sub-cells, kernels and (full load) sub-box shapes and
    capacities for the other strategies, against the oracle."""
    rng = np.random.default_rng(2000 + seed + 31 * ALGOS.index(algo))
    dims = tuple(int(v) for v in rng.integers(3, 13, size=3))
    ppc = float(rng.choice([1, 3, 8, 20]))
    c = synth.scaled_uniform(ppc, dims, seed=300 + seed)
    kernel = ["gaussian", "indicator", "candidate", "lj", "lowflop"][seed % 5]
    xs = int(rng.choice([1, 2, 4]))
    tune = {}
    if algo == "fullload":
        tune = dict(fullload_box=tuple(int(v) for v in rng.integers(1, 6, size=3)),
                    fullload_cap=int(rng.choice([0, 64, 400])))
    want = oracle_interact(c, kernel)
    ctx = ctx_for(c, kernel, x_subcells=xs)
    got, ctx = gpu_interact(c, algo, kernel, tuning=tune, ctx=ctx)
    assert_parity(got, want, label=f"{algo} fuzz {seed} dims {dims} ppc {ppc} sx {xs} {kernel} {tune}")
    assert ctx.stats()["candidates"] == int(want["C"].sum())
