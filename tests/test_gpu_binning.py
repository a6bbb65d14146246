"""a1-a4 parity through the C ABI: cell indices, counts and prefix array bit-exact, M_C exact,
per-cell membership exact as sets, sorted records = bitwise copies of the inputs."""
import json
import os

import numpy as np
import pytest
import torch

import synth
from oracle import celllist
from oracle import reference as ref
from tests._util import ctx_for, to_dev

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def check_binning(cloud, ctx=None):
    if ctx is None:
        ctx = ctx_for(cloud)
    ctx.bin(*to_dev(cloud))
    cell_of, counts, offsets, perm = (t.cpu().numpy().astype(np.int64) for t in ctx.get_binning())
    parts = ctx.get_particles()
    torch.cuda.synchronize()
    g = cloud.grid
    want_cell = celllist.cells(cloud.x, cloud.y, cloud.z, g)
    assert np.array_equal(cell_of, want_cell), "a1 cell index not bit-exact"
    want_counts, want_off, _ = celllist.binning(want_cell, g.ncells)
    assert np.array_equal(counts, want_counts), "a2 counts"
    assert np.array_equal(offsets, want_off), "a3 prefix array"
    assert ref.prefix(want_counts).tolist() == offsets.tolist()
    st = ctx.stats()
    assert st["max_per_cell"] == (int(want_counts.max()) if cloud.n else 0), "M_C"
    # a4: perm is a permutation; every cell segment holds exactly that cell's particles
    assert np.array_equal(np.sort(perm), np.arange(cloud.n))
    seg_cell = np.repeat(np.arange(g.ncells), want_counts)
    assert np.array_equal(want_cell[perm], seg_cell), "membership"
    # sorted records are bitwise copies
    for name, a in (("x", cloud.x), ("y", cloud.y), ("z", cloud.z), ("q", cloud.q)):
        got = parts[name].cpu().numpy()
        assert np.array_equal(got.view(np.uint32), a[perm].view(np.uint32)), name
    assert np.array_equal(parts["id"].cpu().numpy(), perm)
    return ctx


def test_hand2x3():
    g = json.load(open(os.path.join(GOLDEN, "hand2x3.json")))
    c = synth.hand_2x3()
    ctx = check_binning(c)
    _, counts, offsets, perm = ctx.get_binning()
    assert counts.cpu().tolist() == g["counts"]
    assert offsets.cpu().tolist() == g["offsets"]


@pytest.mark.parametrize("name", ["c0", "c1"])
def test_configs(name):
    check_binning(synth.make_config(name))


@pytest.mark.parametrize("n", [0, 1, 2, 3, 5, 4097, 33333])
def test_ragged_sizes(n):
    grid = synth.Grid(dims=(16, 16, 16), w=1 / 16)
    check_binning(synth.uniform(n, grid, seed=77 + n))


def test_scan_tile_edges():
    # Nc around the scan tile (4096) and several tiles with a ragged tail
    for dims in ((16, 16, 16), (17, 16, 16), (15, 16, 17), (64, 64, 3), (1, 1, 1)):
        m = max(dims)
        inv = 1 << int(np.ceil(np.log2(m)))
        grid = synth.Grid(dims=dims, w=1.0 / inv)
        n = 3 * grid.ncells + 7
        c = synth.uniform(n, grid, seed=5)
        check_binning(c)


def test_all_in_one_cell_and_clustered():
    grid = synth.Grid(dims=(8, 8, 8), w=1 / 8)
    rng = np.random.default_rng(3)
    n = 5000
    x = (0.3 + 0.1 * rng.random(n)).astype(np.float32)
    c = synth.Cloud(grid, x, x.copy(), x.copy(), np.ones(n, np.float32))
    check_binning(c)  # all 5000 particles in cell (2, 2, 2)
    check_binning(synth.clustered(200000, synth.Grid(dims=(64, 64, 64), w=1 / 64), seed=9))


def test_nondyadic_grid_contract():
    """C3 with a non-power-of-two width and non-zero origin: bit-exact vs the oracle's fp32 contract."""
    grid = synth.Grid(dims=(7, 5, 3), w=0.1, origin=(0.3, -0.2, 0.05))
    rng = np.random.default_rng(11)
    n = 20000
    x = (rng.random(n) * 0.7 + 0.3).astype(np.float32)
    y = (rng.random(n) * 0.5 - 0.2).astype(np.float32)
    z = (rng.random(n) * 0.3 + 0.05).astype(np.float32)
    check_binning(synth.Cloud(grid, x, y, z, np.ones(n, np.float32)))


def test_rebinning_is_repeatable():
    c = synth.make_config("c0")
    ctx = ctx_for(c)
    for _ in range(3):  # counts are re-zeroed by the scan; the look-back epoch advances
        check_binning(c, ctx)


@pytest.mark.parametrize("kind", ["clustered", "nondyadic"])
def test_partitioned_buckets_with_ids(kind):
    """Random-order pi_bin partitions into buckets of ~2^17 particles before the scatter: cover
    several (uneven) buckets, a non-power-of-two cell count, a ragged tile and caller ids."""
    n = 3 * (1 << 18) + 4101
    if kind == "clustered":
        cloud = synth.clustered(n, synth.Grid(dims=(64, 64, 64), w=1 / 64), seed=31)
    else:
        cloud = synth.uniform(n, synth.Grid(dims=(60, 44, 36), w=1 / 64), seed=32)
    ctx = check_binning(cloud)
    ids = np.random.default_rng(7).permutation(n).astype(np.int32) * 3 + 1
    ctx.bin(*to_dev(cloud), torch.from_numpy(ids).cuda())
    _, _, _, perm = ctx.get_binning()
    parts = ctx.get_particles()
    assert np.array_equal(parts["id"].cpu().numpy(), ids[perm.cpu().numpy()])


def test_cell_sorted_input():
    """pi_bin of input already in cell order (lanes of a warp share cells: the count's
    warp-aggregated atomics add whole runs at once) bins bit-exactly too."""
    c = synth.make_config("c1")
    cells = celllist.cells(c.x, c.y, c.z, c.grid)
    order = np.argsort(cells, kind="stable")
    s = synth.Cloud(c.grid, c.x[order], c.y[order], c.z[order], c.q[order])
    check_binning(s)
