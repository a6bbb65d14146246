"""a8 X-slab decomposition on the GPU, through the C ABI.

P contexts on ONE GPU (the round's boxes have one), linked by the library's in-process
transport ("PILOCAL:<key>"), each driven by its own host thread as one rank per GPU would be.
The exchange kernels (ghost selection, migration, append) and the slab-aware binning and
interaction are the same code the NCCL transport drives; only the byte mover differs.
Checked against the oracle on the WHOLE cloud: per-rank outputs in caller order after
pi_bin, and forces / positions / ownership after each pi_step (migration included)."""
import concurrent.futures as cf
import itertools

import numpy as np
import pytest
import torch

import synth
from oracle import celllist
from oracle import reference as ref
from tests._util import assert_parity

pytestmark = pytest.mark.gpu

_key = itertools.count()


def _contexts(g, P, capacity, kernel="gaussian"):
    from paper_2406_16091_b200 import Context
    uid = f"PILOCAL:test{next(_key)}".encode()
    ctxs = []
    for r in range(P):
        s = torch.cuda.Stream()
        ctxs.append(Context(g.dims, g.w, g.r_c, g.origin, kernel=kernel, sigma=0.0 if g.sigma is None else g.sigma,
                            capacity=capacity, device="cuda", stream=s, rank=r, nranks=P, nccl_unique_id=uid))
    return ctxs


def _all(pool, fn, ctxs):
    futs = [pool.submit(fn, r, c) for r, c in enumerate(ctxs)]
    return [f.result(timeout=120) for f in futs]


def _partition(c, ctx):
    cx = celllist.cells(c.x, c.y, c.z, c.grid) % c.grid.dims[0]
    idx = np.flatnonzero((cx >= ctx.slab["gx_lo"]) & (cx < ctx.slab["gx_hi"]))
    return idx


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("algo", ["global", "xpencil", "fullload", "xpreg", "half"])
def test_slab_bin_interact_matches_whole_cloud(P, algo):
    c = synth.make_config("c0", n=4 * 4096)
    g = c.grid
    ctxs = _contexts(g, P, capacity=c.n)
    parts = [_partition(c, k) for k in ctxs]
    assert sum(len(p) for p in parts) == c.n

    def run(r, k):
        idx = parts[r]
        with torch.cuda.stream(k.stream):
            k.bin(*(_dev(a[idx]) for a in (c.x, c.y, c.z, c.q)), id=_dev(idx.astype(np.int32)))
            out = k.interact(algo)
        k.stream.synchronize()
        return torch.stack(out, 1).cpu().numpy().astype(np.float64), k.stats()

    with cf.ThreadPoolExecutor(P) as pool:
        res = _all(pool, run, ctxs)
    got = np.zeros((c.n, 4))
    for r, (out, st) in enumerate(res):
        got[parts[r]] = out
        assert st["n_owned"] == len(parts[r])
        assert st["fallback_cells"] == 0 or algo == "global"
        if 0 < r < P - 1:
            assert st["n_ghost"] > 0
    want = celllist.interact(c.x, c.y, c.z, c.q, g)
    assert_parity(got, want, label=f"P={P} {algo}")
    # candidate pairs are counted over owned targets only: their sum is the single-domain C
    assert sum(st["candidates"] for _, st in res) == int(want["C"].sum())


def test_slab_binning_counts_exact():
    c = synth.make_config("c0", n=4 * 4096)
    g = c.grid
    P = 2
    ctxs = _contexts(g, P, capacity=c.n)
    parts = [_partition(c, k) for k in ctxs]

    def run(r, k):
        idx = parts[r]
        with torch.cuda.stream(k.stream):
            k.bin(*(_dev(a[idx]) for a in (c.x, c.y, c.z, c.q)))
            counts, offsets = k.get_offsets()
        k.stream.synchronize()
        return counts.cpu().numpy(), offsets.cpu().numpy(), k.slab

    with cf.ThreadPoolExecutor(P) as pool:
        res = _all(pool, run, ctxs)
    gcells = celllist.cells(c.x, c.y, c.z, g)
    wc, _, _ = celllist.binning(gcells, g.ncells)
    wc = wc.reshape(g.dims[2], g.dims[1], g.dims[0])
    for counts, offsets, sl in res:
        nx = sl["nx_local"]
        loc = counts.reshape(g.dims[2], g.dims[1], nx)
        # local X layer j holds global layer gx_off + j (owned and ghost layers alike)
        for j in range(nx):
            gx = sl["gx_off"] + j
            exp = wc[:, :, gx] if 0 <= gx < g.dims[0] else np.zeros_like(loc[:, :, j])
            assert np.array_equal(loc[:, :, j], exp), f"layer {j}"
        assert offsets[-1] == counts.sum()


@pytest.mark.parametrize("algo,P,overlap", [("xpencil", 4, 0), ("xpencil", 2, 0), ("xpencil", 4, 1),
                                             ("xpencil", 2, 1), ("global", 4, 0), ("half", 4, 0)])
def test_slab_steps_migrate_and_match_oracle(algo, P, overlap):
    """Several steps with migration every step.  X-pencil: overlap 0 (default) computes the 2
    boundary layers per side first and exchanges migrants and ghosts on a second stream during
    the interior launch (P = 2: 8 owned layers, an interior launch; P = 4: 4 layers, none);
    overlap 1 exchanges serially at the start of the next step."""
    c = synth.make_config("c0", n=4 * 4096)
    g = c.grid
    ctxs = _contexts(g, P, capacity=c.n)
    for k in ctxs:
        k.set_tuning(exchange_overlap=overlap)
    parts = [_partition(c, k) for k in ctxs]
    # dt so that the fastest particle moves ~0.8 cell per step: migration every step
    F = celllist.interact(c.x, c.y, c.z, c.q, g)["out"][:, 1:]
    dt = float(np.float32(0.8 * g.w / np.abs(F).max()))

    def bin_(r, k):
        idx = parts[r]
        with torch.cuda.stream(k.stream):
            k.bin(*(_dev(a[idx]) for a in (c.x, c.y, c.z, c.q)), id=_dev(idx.astype(np.int32)))

    def state(r, k):
        with torch.cuda.stream(k.stream):
            p = k.get_particles()
        k.stream.synchronize()
        return {key: v.cpu().numpy() for key, v in p.items()}, k.stats()

    def step(r, k):
        with torch.cuda.stream(k.stream):
            k.step(algo, dt)

    def union(states):
        d = {key: np.concatenate([s[key] for s, _ in states]) for key in states[0][0]}
        order = np.argsort(d["id"])
        return {key: v[order] for key, v in d.items()}

    ext = g.extent
    with cf.ThreadPoolExecutor(P) as pool:
        _all(pool, bin_, ctxs)
        s0 = union(_all(pool, state, ctxs))
        assert np.array_equal(s0["id"], np.arange(c.n))
        migrated = 0
        for it in range(3):
            _all(pool, step, ctxs)
            st = _all(pool, state, ctxs)
            s1 = union(st)
            assert np.array_equal(s1["id"], np.arange(c.n)), "a particle lost or duplicated"
            want = celllist.interact(s0["x"], s0["y"], s0["z"], s0["q"], g)
            got = np.stack([s1[k] for k in ("phi", "fx", "fy", "fz")], 1).astype(np.float64)
            assert_parity(got, want, label=f"step {it}")
            for a, ax in enumerate("xyz"):
                exp = ref.integrate(s0[ax], got[:, a + 1], dt, 0.0, ext[a])
                assert np.allclose(s1[ax], exp, rtol=0, atol=2e-7 + 1e-6 * dt)
            ins = sum(s["migrants_in"] for _, s in st)
            outs = sum(s["migrants_out"] for _, s in st)
            assert ins == outs
            migrated += ins
            s0 = s1
        assert migrated > 0
        # the next step re-bins: every rank owns exactly the particles in its slab
        _all(pool, step, ctxs)
        st = _all(pool, state, ctxs)
    for _, stats in st:
        assert stats["overlapped_steps"] == (4 if algo == "xpencil" and overlap == 0 else 0)
    cx = celllist.cells(s0["x"], s0["y"], s0["z"], g) % g.dims[0]
    for r, (s, stats) in enumerate(st):
        sl = ctxs[r].slab
        want_ids = np.flatnonzero((cx >= sl["gx_lo"]) & (cx < sl["gx_hi"]))
        assert np.array_equal(np.sort(s["id"]), want_ids)
    for k in ctxs:
        k.close()


def test_slab_domain_flag():
    """A pi_bin particle outside the rank's slab raises flag 8 (PI_EDEVICE), it is not dropped silently."""
    from paper_2406_16091_b200 import PiError
    c = synth.make_config("c0")
    g = c.grid
    ctxs = _contexts(g, 2, capacity=2 * c.n)

    def run(r, k):
        with torch.cuda.stream(k.stream):
            k.bin(*(_dev(a) for a in (c.x, c.y, c.z, c.q)))  # the whole cloud on both ranks
        k.stream.synchronize()
        try:
            k.stats()
        except PiError as e:
            return str(e)
        return ""

    with cf.ThreadPoolExecutor(2) as pool:
        msgs = _all(pool, run, ctxs)
    assert all("flags 0x8" in m for m in msgs), msgs


def test_slab_exchange_counted_bytes():
    """The two-phase exchange (counts first, then exactly the counted records: SURVEY.md §8(e))
    and the fixed-capacity one (exchange_full = 1) give the same state; the counted one puts only
    the real payload on the links: 20 B per ghost / migrant + a 16-B header per message."""
    c = synth.make_config("c0", n=4 * 4096)
    g = c.grid
    P = 4
    F = celllist.interact(c.x, c.y, c.z, c.q, g)["out"][:, 1:]
    dt = float(np.float32(0.5 * g.w / np.abs(F).max()))
    out = {}
    for full in (0, 1):
        ctxs = _contexts(g, P, capacity=c.n)
        parts = [_partition(c, k) for k in ctxs]

        def run(r, k):
            k.set_tuning(exchange_full=full)
            idx = parts[r]
            with torch.cuda.stream(k.stream):
                k.bin(*(_dev(a[idx]) for a in (c.x, c.y, c.z, c.q)), id=_dev(idx.astype(np.int32)))
                k.step("xpencil", dt)
                p = k.get_particles()
            k.stream.synchronize()
            return {key: v.cpu().numpy() for key, v in p.items()}, k.stats()

        with cf.ThreadPoolExecutor(P) as pool:
            out[full] = _all(pool, run, ctxs)
        for k in ctxs:
            k.close()
    for full in (0, 1):
        ids = np.concatenate([s["id"] for s, _ in out[full]])
        assert np.array_equal(np.sort(ids), np.arange(c.n))
    for r in range(P):
        (s0, st0), (s1, st1) = out[0][r], out[1][r]
        o0, o1 = np.argsort(s0["id"]), np.argsort(s1["id"])
        assert np.array_equal(s0["id"][o0], s1["id"][o1])
        for key in ("x", "y", "z", "phi", "fx", "fy", "fz"):  # (sums in another order after the atomic scatter)
            a, b = s0[key][o0].astype(np.float64), s1[key][o1].astype(np.float64)
            assert np.allclose(a, b, rtol=1e-5, atol=1e-5 * np.abs(b).max()), key
        nmsg = 3 * ((r > 0) + (r < P - 1))  # pi_bin's ghost exchange + the step's migration and ghosts
        assert st0["exchange_bytes"] >= 20 * st0["migrants_out"] + 16 * nmsg
        assert st0["exchange_bytes"] < st1["exchange_bytes"] / 2  # the counted records, not the capacity


def test_slab_overlap_larger_sampled():
    """The overlapped step at a size with real interior launches and large messages: 2^20 uniform
    particles on 64^3 cells, P = 4 (16 owned layers per rank), two steps with migration, sampled
    targets against the oracle on the whole cloud of the pre-step state; the serial exchange
    gives the same state."""
    c = synth.scaled_uniform(4, (64, 64, 64), seed=240616099)
    g = c.grid
    P = 4
    F = celllist.interact(c.x, c.y, c.z, c.q, g, targets=np.arange(0, c.n, 97))["out"][:, 1:]
    dt = float(np.float32(0.4 * g.w / np.abs(F).max()))
    res = {}
    for overlap in (0, 1):
        ctxs = _contexts(g, P, capacity=c.n)
        parts = [_partition(c, k) for k in ctxs]

        def run(r, k):
            k.set_tuning(exchange_overlap=overlap)
            idx = parts[r]
            with torch.cuda.stream(k.stream):
                k.bin(*(_dev(a[idx]) for a in (c.x, c.y, c.z, c.q)), id=_dev(idx.astype(np.int32)))
                k.step("xpencil", dt)
                p0 = k.get_particles()
                k.step("xpencil", dt)
                p1 = k.get_particles()
            k.stream.synchronize()
            return ({key: v.cpu().numpy() for key, v in p0.items()}, {key: v.cpu().numpy() for key, v in p1.items()},
                    k.stats())

        with cf.ThreadPoolExecutor(P) as pool:
            out = _all(pool, run, ctxs)
        for k in ctxs:
            k.close()
        res[overlap] = out
        for _, _, st in out:
            assert st["overlapped_steps"] == (2 if overlap == 0 else 0)

    def union(states):
        d = {key: np.concatenate([s[key] for s in states]) for key in states[0]}
        order = np.argsort(d["id"])
        return {key: v[order] for key, v in d.items()}

    for overlap in (0, 1):
        s0 = union([o[0] for o in res[overlap]])
        s1 = union([o[1] for o in res[overlap]])
        assert np.array_equal(s1["id"], np.arange(c.n)), "a particle lost or duplicated"
        sample = np.random.default_rng(3).choice(c.n, 4000, replace=False)
        want = celllist.interact(s0["x"], s0["y"], s0["z"], s0["q"], g, targets=sample)
        got = np.stack([s1[k][sample] for k in ("phi", "fx", "fy", "fz")], 1).astype(np.float64)
        assert_parity(got, want, label=f"overlap={overlap} step 2")
    # after the first step both modes hold the same state up to the forces' summation order (the
    # second step can differ more: pairs at r ~ r_c may fall on either side after such changes)
    a, b = union([o[0] for o in res[0]]), union([o[0] for o in res[1]])
    for key in ("x", "y", "z"):
        assert np.allclose(a[key], b[key], rtol=0, atol=1e-6)


@pytest.mark.parametrize("seed", range(6))
def test_slab_fuzz(seed):
    """Random X-slab runs: grid, density, P (dividing dims[0]), strategy, overlapped or serial and
    two-phase or fixed-capacity exchange, two steps with migration; the union of the ranks' owned
    particles is checked against the whole-cloud oracle after every step."""
    rng = np.random.default_rng(4000 + seed)
    nx = int(rng.choice([8, 12, 16]))
    P = int(rng.choice([d for d in (2, 3, 4) if nx % d == 0]))
    dims = (nx, int(rng.integers(3, 9)), int(rng.integers(3, 9)))
    ppc = float(rng.choice([2, 6, 12]))
    c = synth.scaled_uniform(ppc, dims, seed=500 + seed)
    g = c.grid
    algo = ["xpencil", "global", "half"][seed % 3]
    tune = dict(exchange_overlap=int(rng.integers(0, 2)), exchange_full=int(rng.integers(0, 2)))
    F = celllist.interact(c.x, c.y, c.z, c.q, g)["out"][:, 1:]
    dt = float(np.float32(0.7 * g.w / np.abs(F).max()))
    ctxs = _contexts(g, P, capacity=c.n)
    parts = [_partition(c, k) for k in ctxs]

    def run(r, k):
        k.set_tuning(**tune)
        idx = parts[r]
        states = []
        with torch.cuda.stream(k.stream):
            k.bin(*(_dev(a[idx]) for a in (c.x, c.y, c.z, c.q)), id=_dev(idx.astype(np.int32)))
            for _ in range(2):
                k.step(algo, dt)
                states.append({key: v.cpu().numpy() for key, v in k.get_particles().items()})
        k.stream.synchronize()
        return states, k.stats()

    with cf.ThreadPoolExecutor(P) as pool:
        res = _all(pool, run, ctxs)
    for k in ctxs:
        k.close()

    def union(states):
        d = {key: np.concatenate([s[key] for s in states]) for key in states[0]}
        order = np.argsort(d["id"])
        return {key: v[order] for key, v in d.items()}

    prev = {"x": c.x, "y": c.y, "z": c.z, "q": c.q}
    for it in range(2):
        s1 = union([st[it] for st, _ in res])
        assert np.array_equal(s1["id"], np.arange(c.n)), "a particle lost or duplicated"
        want = celllist.interact(prev["x"], prev["y"], prev["z"], prev["q"], g)
        got = np.stack([s1[k] for k in ("phi", "fx", "fy", "fz")], 1).astype(np.float64)
        assert_parity(got, want, label=f"slab fuzz {seed} P={P} dims={dims} {algo} {tune} step {it}")
        prev = s1
    for _, st in res:
        ovl = algo == "xpencil" and tune["exchange_overlap"] == 0 and nx // P >= 4
        assert st["overlapped_steps"] == (2 if ovl else 0)


def test_slab_run_host():
    """pi_run_host with X-slabs (the e2e path of bench.py at N > 1): each rank passes its slab's
    particles in pinned host memory and gets its outputs back in caller order."""
    c = synth.make_config("c0", n=4 * 4096)
    g = c.grid
    P = 2
    ctxs = _contexts(g, P, capacity=c.n)
    parts = [_partition(c, k) for k in ctxs]

    def run(r, k):
        idx = parts[r]
        h = [torch.from_numpy(np.ascontiguousarray(a[idx])).pin_memory() for a in (c.x, c.y, c.z, c.q)]
        o = [torch.empty(len(idx), dtype=torch.float32).pin_memory() for _ in range(4)]
        with torch.cuda.stream(k.stream):
            k.run_host("xpencil", *h, *o)
            k.run_host("xpencil", *h, *o)  # twice: the second reuses the context's state
        k.stream.synchronize()
        return torch.stack(o, 1).numpy().astype(np.float64)

    with cf.ThreadPoolExecutor(P) as pool:
        res = _all(pool, run, ctxs)
    for k in ctxs:
        k.close()
    got = np.zeros((c.n, 4))
    for r in range(P):
        got[parts[r]] = res[r]
    assert_parity(got, celllist.interact(c.x, c.y, c.z, c.q, g), label="slab run_host")
