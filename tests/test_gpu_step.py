"""pi_step (a1-a7): one step = bin, interact, x <- x + dt F (reflecting walls).  Checked one step
at a time against the oracle applied to the GPU's pre-step state (C11), never as free-running
trajectories; the re-binning of the updated positions is checked bit-exact."""
import numpy as np
import pytest
import torch

import synth
from oracle import celllist
from oracle import reference as ref
from tests._util import KERNEL_ID, assert_parity, ctx_for, to_dev

pytestmark = pytest.mark.gpu


def state(ctx):
    p = ctx.get_particles()
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in p.items()}


@pytest.mark.parametrize("algo,kernel,xs,tune", [("global", "gaussian", 0, None), ("xpencil", "gaussian", 0, None),
                                                  ("fullload", "gaussian", 0, None), ("xpencil", "gaussian", 1, None),
                                                  ("xpencil", "gaussian", 8, None), ("xpencil", "lj", 0, None),
                                                  ("global", "lj", 4, None), ("xpreg", "gaussian", 2, None),
                                                  ("half", "gaussian", 0, None), ("half", "lj", 2, None),
                                                  # every cell through the Par-Cell-SM pass
                                                  ("xpencil", "gaussian", 0, dict(xpencil_cap=16)),
                                                  ("xpencil", "lj", 2, dict(xpencil_cap=16)),
                                                  # the interleaved staging (records, not pairs)
                                                  ("xpencil", "gaussian", 4, dict(xpencil_layout=1))])
def test_step_matches_oracle(algo, kernel, xs, tune):
    """Three steps, each checked against the oracle at the GPU's pre-step state; the re-binning
    (counts carried by the update, R18 sub-cells) must be bit-exact per cell afterwards."""
    c = synth.make_config("c0")
    g = c.grid
    ctx = ctx_for(c, kernel, x_subcells=xs)
    if tune:
        ctx.set_tuning(**tune)
    ctx.bin(*to_dev(c))
    s0 = state(ctx)                                   # sorted state before the step
    # dt: a few % of the particles change sub-cell each step (the Gaussian forces of c0 are
    # ~1e2, LJ's ~1e4)
    dt = np.float32(1e-5 if kernel == "gaussian" else 1e-7)
    for it in range(3):
        ctx.step(algo, float(dt))
        s1 = state(ctx)                               # updated positions + this step's outputs
        # forces of this step vs the oracle at the pre-step positions (matched by id)
        order0 = np.argsort(s0["id"])
        order1 = np.argsort(s1["id"])
        X0 = [s0[k][order0] for k in ("x", "y", "z", "q")]
        want = celllist.interact(*X0, g, kernel=KERNEL_ID[kernel])
        got = np.stack([s1[k][order1] for k in ("phi", "fx", "fy", "fz")], 1).astype(np.float64)
        assert_parity(got, want, label=f"step{it} forces")
        # position update: x + dt F, reflected, from the GPU's own forces (fp32 fma -> 1 ulp)
        for ax, f in (("x", "fx"), ("y", "fy"), ("z", "fz")):
            exp = ref.integrate(s0[ax][order0], got[:, "xyz".index(ax) + 1], float(dt), 0.0, 1.0)
            assert np.allclose(s1[ax][order1], exp, rtol=0, atol=2e-7 + 1e-6 * float(dt))
        # re-binning of the updated positions is bit-exact (checked on the next binning)
        s0 = s1
    counts, offsets = ctx.get_offsets()
    ctx.step(algo, float(dt))      # bins s0 (= last updated positions) before interacting
    counts, offsets = (t.cpu().numpy() for t in ctx.get_offsets())
    cells = celllist.cells(s0["x"], s0["y"], s0["z"], g)
    wc, wo, _ = celllist.binning(cells, g.ncells)
    assert np.array_equal(counts, wc) and np.array_equal(offsets, wo)
    assert ctx.stats()["steps"] == 4


def test_step_capturable_in_cuda_graph():
    """pi_step does no allocation and no host synchronisation (include/pi.h): a step captured in a
    CUDA graph and replayed gives the same state as the same steps run eagerly."""
    c = synth.make_config("c0")
    dt = 1e-5
    s = torch.cuda.Stream()
    eager = ctx_for(c, stream=s)
    graphed = ctx_for(c, stream=s)
    with torch.cuda.stream(s):
        for k in (eager, graphed):
            k.bin(*to_dev(c))
            k.step("xpencil", dt)          # first step reuses pi_bin's binning
        eager.step("xpencil", dt)
        eager.step("xpencil", dt)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            graphed.step("xpencil", dt)    # re-bin + interact + update, captured
        g.replay()
        g.replay()
    s.synchronize()
    a, b = state(eager), state(graphed)
    oa, ob = np.argsort(a["id"]), np.argsort(b["id"])
    assert np.array_equal(a["id"][oa], b["id"][ob])
    for key in ("x", "y", "z"):  # same arithmetic; within-cell order (atomics) may differ
        assert np.allclose(a[key][oa], b[key][ob], rtol=0, atol=1e-6)


@pytest.mark.parametrize("name,steps", [("c1", 3), ("c4", 2)])
def test_step_full_size_sampled(name, steps):
    """pi_step in the bench's configuration (the X-pencil, default tuning, the carried-count
    re-binning of the nearly sorted records, the fused update) at configs[1] (2^21, 64^3) and
    configs[4] (2^27, 256^3): after warm-up steps, one step's forces on sampled particles against
    the oracle at the GPU's pre-step state (C11), the update against x + dt F, and the following
    re-binning bit-exact per cell against the oracle's binning of the updated positions."""
    c = synth.make_config(name)
    g = c.grid
    ctx = ctx_for(c)
    ctx.bin(*to_dev(c))
    _, fx, fy, fz = ctx.interact("xpencil")
    fmax = float(torch.stack([fx.abs().max(), fy.abs().max(), fz.abs().max()]).max())
    dt = float(np.float32(0.01 * g.w / fmax))   # max |dx| = 1 % of a cell per step
    for _ in range(steps):
        ctx.step("xpencil", dt)
    s0 = state(ctx)
    ctx.step("xpencil", dt)
    s1 = state(ctx)
    order0, order1 = np.argsort(s0["id"]), np.argsort(s1["id"])
    assert np.array_equal(s0["id"][order0], s1["id"][order1])
    X0 = [s0[k][order0] for k in ("x", "y", "z", "q")]
    sample = np.random.default_rng(11).choice(c.n, 3000, replace=False)
    want = celllist.interact(*X0, g, targets=sample)
    got = np.stack([s1[k][order1][sample] for k in ("phi", "fx", "fy", "fz")], 1).astype(np.float64)
    assert_parity(got, want, label=f"{name} step forces")
    for ax, a in (("x", 1), ("y", 2), ("z", 3)):
        exp = ref.integrate(X0["xyz".index(ax)][sample], got[:, a], dt, 0.0, 1.0)
        assert np.allclose(s1[ax][order1][sample], exp, rtol=0, atol=2e-7 + 1e-6 * dt)
    moved = np.mean(celllist.cells(s1["x"], s1["y"], s1["z"], g) != celllist.cells(s0["x"], s0["y"], s0["z"], g))
    assert moved > 0   # the step moved particles across cells: the re-binning below is exercised
    ctx.step("xpencil", dt)    # re-bins s1's positions before interacting
    counts, offsets = (t.cpu().numpy() for t in ctx.get_offsets())
    wc, wo, _ = celllist.binning(celllist.cells(s1["x"], s1["y"], s1["z"], g), g.ncells)
    assert np.array_equal(counts, wc) and np.array_equal(offsets, wo)
