"""X-slab decomposition (north star row a8) on CPU, world_size 2 over `gloo` (-m "not gpu").

The library's exchange runs on the GPU; what is checked here is the host-side contract it
relies on, with real ranks and a real transport:
  * pi_slab_info (the library's own host logic) tiles the global X range, one slab per rank,
    with one ghost layer on each side;
  * the protocol -- each rank sends its first / last owned X layer as ghosts, interacts its
    owned targets against owned + ghost sources -- reproduces the single-domain result
    (the oracle on the whole cloud), because cell_width >= r_c makes one ghost
    layer enough;
  * migration after a position update (|dx| < w) keeps every particle owned exactly once,
    by the rank whose slab holds its new cell;
  * the overlapped step's selection (migrants and next ghosts taken from the first / last 2
    owned layers plus the arrivals) gives the serial protocol's ghost sets.
Ghost and migrant messages are exchanged with torch.distributed send/recv between two real
processes; the interactions are the oracle's."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import celllist
from oracle import reference as ref

WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _send_arrays(arrs, dst):
    n = torch.tensor([len(arrs[0])], dtype=torch.int64)
    dist.send(n, dst)
    for a in arrs:
        if len(a):
            dist.send(torch.from_numpy(np.ascontiguousarray(a)), dst)


def _recv_arrays(dtypes, src):
    n = torch.zeros(1, dtype=torch.int64)
    dist.recv(n, src)
    out = []
    for dt in dtypes:
        t = torch.empty(int(n.item()), dtype=dt)
        if len(t):
            dist.recv(t, src)
        out.append(t.numpy())
    return out


def _exchange(rank, send_left, send_right, dtypes):
    """Blocking neighbour exchange in an order that cannot deadlock (even ranks send first)."""
    got = []
    for phase in (0, 1):
        for nb, payload in ((rank - 1, send_left), (rank + 1, send_right)):
            if not 0 <= nb < WORLD:
                continue
            if (rank + phase) % 2 == 0:
                _send_arrays(payload, nb)
            else:
                got.append((nb, _recv_arrays(dtypes, nb)))
    return got


def _worker(rank, port, result_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=WORLD)
    try:
        from paper_2406_16091_b200 import slab_info
        c = synth.make_config("c0", n=4 * 4096)  # 4 particles per cell on 16^3, same cloud on every rank
        g = c.grid
        info = slab_info(g.dims, g.w, rank, WORLD, capacity=c.n, r_c=g.r_c)
        lo, hi = info["gx_lo"], info["gx_hi"]
        # the slabs tile [0, dims[0]) in rank order
        spans = [None] * WORLD
        dist.all_gather_object(spans, (lo, hi))
        assert spans[0][0] == 0 and spans[-1][1] == g.dims[0]
        assert all(spans[k][1] == spans[k + 1][0] for k in range(WORLD - 1))
        assert info["nx_local"] == hi - lo + 2 and info["own_lo"] == 1 and info["own_hi"] == hi - lo + 1
        assert info["gx_off"] == lo - 1

        ids = np.arange(c.n, dtype=np.int32)
        cx = celllist.cells(c.x, c.y, c.z, g) % g.dims[0]
        mine = (cx >= lo) & (cx < hi)
        own = [a[mine] for a in (c.x, c.y, c.z, c.q)] + [ids[mine]]
        ocx = cx[mine]

        # ghosts: first owned layer -> rank - 1, last owned layer -> rank + 1
        fl, ll = ocx == lo, ocx == hi - 1
        dtypes = (torch.float32,) * 4 + (torch.int32,)
        got = _exchange(rank, [a[fl] for a in own], [a[ll] for a in own], dtypes)
        ghosts = [np.concatenate([own[k][:0]] + [p[k] for _, p in got]) for k in range(5)]
        gcx = celllist.cells(ghosts[0], ghosts[1], ghosts[2], g) % g.dims[0]
        assert np.all((gcx == lo - 1) | (gcx == hi)), "a ghost outside the ghost layers"

        # owned targets against owned + ghost sources == the whole-cloud result
        src = [np.concatenate([own[k], ghosts[k]]) for k in range(5)]
        n_own = len(own[0])
        local = celllist.interact(*src[:4], g, targets=np.arange(n_own))
        whole = celllist.interact(c.x, c.y, c.z, c.q, g, targets=np.flatnonzero(mine))
        assert np.array_equal(local["C"], whole["C"]) and np.array_equal(local["P"], whole["P"])
        np.testing.assert_allclose(local["out"], whole["out"], rtol=1e-12, atol=1e-12 * np.abs(whole["S"]).max())
        ind_l = celllist.interact(*src[:4], g, kernel=ref.KERNEL_INDICATOR, targets=np.arange(n_own))
        ind_w = celllist.interact(c.x, c.y, c.z, c.q, g, kernel=ref.KERNEL_INDICATOR, targets=np.flatnonzero(mine))
        assert np.array_equal(ind_l["P"], ind_w["P"])

        # migration: x <- x + dt F with |dt F| < w, then owned particles leaving the slab move
        f = local["out"][:, 1:]
        dt = 0.9 * g.w / max(np.abs(f).max(), 1e-30)
        ext = g.extent
        new = [ref.integrate(own[a].astype(np.float64), f[:, a], dt, 0.0, ext[a]).astype(np.float32)
               for a in range(3)]
        new_state = new + [own[3], own[4]]
        ncx = celllist.cells(new[0], new[1], new[2], g) % g.dims[0]
        assert np.all(np.abs(ncx - ocx) <= 1)
        go_l, go_r, stay = ncx < lo, ncx >= hi, (ncx >= lo) & (ncx < hi)
        got = _exchange(rank, [a[go_l] for a in new_state], [a[go_r] for a in new_state], dtypes)
        after = [np.concatenate([new_state[k][stay]] + [p[k] for _, p in got]) for k in range(5)]
        acx = celllist.cells(after[0], after[1], after[2], g) % g.dims[0]
        assert np.all((acx >= lo) & (acx < hi))
        moved = int(go_l.sum() + go_r.sum())

        # the overlapped step (pi_tuning.exchange_overlap) takes the migrants and
        # the next step's ghosts from the particles of the first / last 2 owned layers (their
        # old cells) plus the arrivals: with |dt F| < w that is every leaver and every particle
        # that ends in a boundary layer, so its ghost messages equal the serial protocol's
        # (the first / last owned layer of the state after migration)
        bnd = (ocx < lo + 2) | (ocx >= hi - 2)
        assert not np.any((go_l | go_r) & ~bnd), "a leaver outside the boundary layers"
        arr_ids = np.concatenate([p[4] for _, p in got]) if got else np.zeros(0, np.int32)
        arr_cx = (celllist.cells(*[np.concatenate([p[k] for _, p in got]) for k in range(3)], g) % g.dims[0]
                  if len(arr_ids) else np.zeros(0, np.int64))
        for side, layer in (("L", lo), ("R", hi - 1)):
            serial = np.sort(after[4][acx == layer])
            ovl = np.sort(np.concatenate([own[4][bnd & stay & (ncx == layer)], arr_ids[arr_cx == layer]]))
            assert np.array_equal(serial, ovl), f"overlapped ghost set differs ({side})"
        all_ids = [None] * WORLD
        dist.all_gather_object(all_ids, (after[4].tolist(), moved))
        if rank == 0:
            flat = np.concatenate([np.asarray(a, np.int64) for a, _ in all_ids])
            assert np.array_equal(np.sort(flat), np.arange(c.n)), "a particle lost or duplicated"
            assert sum(m for _, m in all_ids) > 0, "the step moved nobody across the slab face"
            open(os.path.join(result_dir, "ok"), "w").write("ok")
    finally:
        dist.destroy_process_group()


def test_slab_protocol_gloo_world2(tmp_path):
    from paper_2406_16091_b200 import build
    build.build()
    mp.spawn(_worker, args=(_free_port(), str(tmp_path)), nprocs=WORLD, join=True)
    assert (tmp_path / "ok").exists()


def test_slab_info_tiles_and_validates():
    from paper_2406_16091_b200 import PiError, build, slab_info
    build.build()
    for P in (1, 2, 4, 8):
        spans = [slab_info((64, 8, 8), 1 / 64, r, P, capacity=1 << 16) for r in range(P)]
        assert [s["gx_lo"] for s in spans] == [r * 64 // P for r in range(P)]
        assert all(s["gx_hi"] - s["gx_lo"] == 64 // P for s in spans)
        if P == 1:
            assert spans[0]["nx_local"] == 64 and spans[0]["own_lo"] == 0 and spans[0]["msg_cap"] == 0
        else:
            assert all(s["nx_local"] == 64 // P + 2 and s["msg_cap"] > 0 for s in spans)
    with pytest.raises(PiError):
        slab_info((16, 8, 8), 1 / 16, 0, 3)  # dims[0] % nranks
    with pytest.raises(PiError):
        slab_info((16, 8, 8), 1 / 16, 2, 2)  # rank >= nranks
