"""pi_bin, then a few pi_step calls on one config (for ncu capture of the re-binning kernels:
-k regex:"k_scan|k_scatter" -s 4 -c 2 skips pi_bin and the first step)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2406_16091_b200 import Context
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2_ppc8"
c = synth.make_config(cfg); g = c.grid
ctx = Context(g.dims, g.w, g.r_c, g.origin, capacity=c.n)
t = [torch.from_numpy(v).cuda() for v in (c.x, c.y, c.z, c.q)]
ctx.bin(*t)
_, fx, fy, fz = ctx.interact("xpencil")
dt = 0.01 * g.w / float(torch.stack([fx.abs().max(), fy.abs().max(), fz.abs().max()]).max())
for _ in range(3):
    ctx.step("xpencil", dt)
torch.cuda.synchronize()
print("done")
