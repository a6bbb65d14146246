import sys, os
sys.path.insert(0, '/root/repo')
import torch, synth
from paper_2406_16091_b200 import Context
for xs in (1, 2, 4):
    c = synth.scaled_uniform(64, (12, 10, 9), seed=240616093 + 64)
    g = c.grid
    ctx = Context(g.dims, g.w, g.r_c, g.origin, capacity=c.n, x_subcells=xs)
    t = [torch.from_numpy(v).cuda() for v in (c.x, c.y, c.z, c.q)]
    ctx.bin(*t)
    try:
        ctx.interact("xpencil"); torch.cuda.synchronize(); print(xs, "ok", ctx.stats()["fallback_cells"])
    except Exception as e:
        print(xs, "ERR", e)
