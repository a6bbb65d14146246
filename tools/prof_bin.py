"""pi_bin on random-order input a few times (for ncu capture of the binning kernels)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2406_16091_b200 import Context
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2_ppc8"
c = synth.make_config(cfg); g = c.grid
ctx = Context(g.dims, g.w, g.r_c, g.origin, capacity=c.n)
t = [torch.from_numpy(v).cuda() for v in (c.x, c.y, c.z, c.q)]
for _ in range(3):
    ctx.bin(*t)
torch.cuda.synchronize()
print("done")
