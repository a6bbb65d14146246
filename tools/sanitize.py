"""Small end-to-end run of every kernel of the library for compute-sanitizer (memcheck, racecheck,
synccheck, initcheck): pi_bin of random-order input, pi_interact with every strategy and kernel,
pi_step (carried-count re-binning), the dense-cell (Par-Cell-SM) path, on configs[0] and a
clustered 2^16 cloud.  usage: compute-sanitizer --tool T python tools/sanitize.py"""
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
        for algo in ("global", "fullload", "xpencil"):
            ctx.interact(algo)
        ctx.set_tuning(xpencil_cap=64)  # lists cells for the Par-Cell-SM pass
        ctx.interact("xpencil")
        ctx.set_tuning()
        if kernel == "gaussian":
            for algo in ("xpencil", "global", "fullload"):
                ctx.step(algo, 1e-6)
        torch.cuda.synchronize()
        ctx.close()
print("sanitize run done")
