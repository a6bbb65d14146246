"""bin + interact on one config with tuning from a JSON argument (for ncu captures; development aid).
usage: python tools/prof_tune.py CONFIG 'JSON tuning' [reps]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2406_16091_b200 import Context
c = synth.make_config(sys.argv[1]); g = c.grid
ctx = Context(g.dims, g.w, g.r_c, g.origin, capacity=c.n)
tune = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
if tune: ctx.set_tuning(**tune)
t = [torch.from_numpy(v).cuda() for v in (c.x, c.y, c.z, c.q)]
for _ in range(int(sys.argv[3]) if len(sys.argv) > 3 else 3):
    ctx.bin(*t)
    ctx.interact("xpencil", out=False)
torch.cuda.synchronize()
print("done")
