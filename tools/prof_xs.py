"""bin + interact with a given x_subcells (ncu capture helper)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2406_16091_b200 import Context
xs = int(sys.argv[1]) if len(sys.argv) > 1 else 4
c = synth.make_config("c1"); g = c.grid
ctx = Context(g.dims, g.w, g.r_c, g.origin, capacity=c.n, x_subcells=xs)
t = [torch.from_numpy(v).cuda() for v in (c.x, c.y, c.z, c.q)]
for _ in range(3):
    ctx.bin(*t)
    ctx.interact("xpencil", out=False)
torch.cuda.synchronize()
