"""bin + interact on one config with a chosen libpi build (for ncu A/B captures; development aid).
usage: LIBPI=path python tools/prof_lib.py CONFIG ALGO REPS [JSON tuning] (XSUB env: x_subcells)"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_16091_b200._lib as _L
if os.environ.get("LIBPI"):
    _L.LIBPATH = os.path.abspath(os.environ["LIBPI"])
import torch, synth
from paper_2406_16091_b200 import Context
cfg, algo, reps = sys.argv[1], sys.argv[2], int(sys.argv[3])
tune = json.loads(sys.argv[4]) if len(sys.argv) > 4 else {}
c = synth.make_config(cfg); g = c.grid
ctx = Context(g.dims, g.w, g.r_c, g.origin, capacity=c.n, x_subcells=int(os.environ.get("XSUB", "0")))
if tune: ctx.set_tuning(**tune)
t = [torch.from_numpy(v).cuda() for v in (c.x, c.y, c.z, c.q)]
for _ in range(reps):
    ctx.bin(*t)
    ctx.interact(algo, out=False)
torch.cuda.synchronize()
print("done")
