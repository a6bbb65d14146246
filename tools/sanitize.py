"""Small end-to-end run of every kernel of the library for compute-sanitizer (memcheck, racecheck,
synccheck, initcheck): pi_bin of random-order input, pi_interact with every strategy and kernel,
pi_step (carried-count re-binning), the dense-cell (Par-Cell-SM) path, on configs[0] and a
clustered 2^16 cloud; then X-slabs: 2 contexts on one GPU (in-process transport, one host
thread each), pi_bin + three pi_step with the overlapped exchange and with the serial one.  usage: compute-sanitizer --tool T python tools/sanitize.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
from paper_2406_16091_b200 import Context

clouds = [synth.make_config("c0"), synth.clustered(1 << 16, synth.Grid(dims=(24, 24, 24), w=1 / 24), seed=5)]
for c in clouds:
    g = c.grid
    t = [torch.from_numpy(v).cuda() for v in (c.x, c.y, c.z, c.q)]
    for kernel in ("gaussian", "indicator", "candidate", "lj", "lowflop", "highflop"):
        lj = (g.lj_ref, g.lj_soft, g.lj_e0) if kernel in ("lj", "highflop") else (0, 0, 0)
        ctx = Context(g.dims, g.w, g.r_c, g.origin, kernel=kernel, capacity=c.n, lj=lj)
        ctx.bin(*t)
        for algo in ("global", "fullload", "xpencil", "xpreg", "half"):
            ctx.interact(algo)
        ctx.set_tuning(xpencil_cap=64)  # lists cells for the Par-Cell-SM pass
        ctx.interact("xpencil")
        ctx.set_tuning()
        if kernel == "gaussian":
            for algo in ("xpencil", "global", "fullload", "half"):
                ctx.step(algo, 1e-6)
        torch.cuda.synchronize()
        ctx.close()

# X-slabs (a8): P = 2, 8 owned layers each (an interior launch), migration every step
import concurrent.futures as cf
import numpy as np
c = synth.make_config("c0", n=4 * 4096)
g = c.grid
for overlap in (0, 1):
    uid = f"PILOCAL:sanitize{overlap}".encode()
    ctxs = [Context(g.dims, g.w, g.r_c, g.origin, capacity=c.n, stream=torch.cuda.Stream(), rank=r, nranks=2,
                    nccl_unique_id=uid) for r in range(2)]
    cx = (c.x * g.dims[0]).astype(np.int64)

    def run(r, k):
        k.set_tuning(exchange_overlap=overlap)
        idx = np.flatnonzero((cx >= k.slab["gx_lo"]) & (cx < k.slab["gx_hi"]))
        with torch.cuda.stream(k.stream):
            k.bin(*(torch.from_numpy(np.ascontiguousarray(a[idx])).cuda() for a in (c.x, c.y, c.z, c.q)),
                  id=torch.from_numpy(idx.astype(np.int32)).cuda())
            for _ in range(3):
                k.step("xpencil", 2e-6)
            k.get_particles()
        k.stream.synchronize()
        return k.stats()["overlapped_steps"]

    with cf.ThreadPoolExecutor(2) as pool:
        print("slabs overlap", overlap, [f.result(timeout=600) for f in [pool.submit(run, r, k) for r, k in enumerate(ctxs)]])
    for k in ctxs:
        k.close()
print("sanitize run done")
