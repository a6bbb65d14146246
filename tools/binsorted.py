import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth
from oracle import celllist
from paper_2406_16091_b200 import Context
for name in ("c2_ppc8",):
    c = synth.make_config(name); g = c.grid
    order = np.argsort(celllist.cells(c.x, c.y, c.z, g), kind="stable")
    for label, idx in (("random", np.arange(c.n)), ("sorted", order)):
        t = [torch.from_numpy(np.ascontiguousarray(v[idx])).cuda() for v in (c.x, c.y, c.z, c.q)]
        ctx = Context(g.dims, g.w, g.r_c, g.origin, capacity=c.n)
        ms = []
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        for r in range(8):
            flush.zero_()
            ctx.bin(*t); torch.cuda.synchronize()
            ms.append(ctx.stats()["bin_ms"])
        print(name, label, "pi_bin ms", sorted(ms)[4])
        ctx.close()
