import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_16091_b200._lib as L
L.LIBPATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpi_prof.so")
import torch, synth
from paper_2406_16091_b200 import Context
c = synth.make_config("c1"); g = c.grid
ctx = Context(g.dims, g.w, g.r_c, g.origin, capacity=c.n)
t = [torch.from_numpy(v).cuda() for v in (c.x, c.y, c.z, c.q)]
ctx.bin(*t)
lib = L.load()
buf = (ctypes.c_ulonglong * 16)()
for tune in ({}, {"xpencil_len": 64}, {"threads": 512}):
    ctx.set_tuning(**tune)
    ctx.interact("xpencil", out=False); torch.cuda.synchronize()
    lib.pi_debug_xp_profile(buf)
    ctx.interact("xpencil", out=False); torch.cuda.synchronize()
    lib.pi_debug_xp_profile(buf)
    v = list(buf)
    items = 8192 if not tune.get("xpencil_len") else 4096
    names = ["prod wait empty", "prod tables", "prod stage_round", "prod cp.async wait", "prod stage->arrive", "prod total", "cons wait full", "cons compute", "cons warp-items"]
    print(tune)
    for i, n in enumerate(names):
        print(f"  {n:22s} {v[i]:16d}  per item {v[i]/items:12.0f}")
