"""Run bin + interact on one config a few times (for ncu capture)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2406_16091_b200 import Context
cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
algo = sys.argv[2] if len(sys.argv) > 2 else "xpencil"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
c = synth.make_config(cfg)
g = c.grid
ctx = Context(g.dims, g.w, g.r_c, g.origin, capacity=c.n, x_subcells=int(os.environ.get("XSUB", "0")))
if os.environ.get('TPL') or os.environ.get('TGT') or os.environ.get('THREADS') or os.environ.get('LEN'):
    ctx.set_tuning(xpencil_slots=int(os.environ.get('TPL', '0')), xpencil_targets=int(os.environ.get('TGT', '0')),
                   threads=int(os.environ.get('THREADS', '0')), xpencil_len=int(os.environ.get('LEN', '0')))
t = [torch.from_numpy(v).cuda() for v in (c.x, c.y, c.z, c.q)]
for _ in range(reps):
    ctx.bin(*t)
    ctx.interact(algo, out=False)
torch.cuda.synchronize()
print("done")
