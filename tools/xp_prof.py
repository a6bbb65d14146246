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
mode = int(sys.argv[1]) if len(sys.argv) > 1 else 0
# (no modes)
for tune in ({}, {"xpencil_len": 32}):
    ctx.set_tuning(**tune)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ctx.interact("xpencil", out=False)
    e1.record(); torch.cuda.synchronize()
    print("mode", mode, tune, "kernel ms", e0.elapsed_time(e1))
    ctx.interact("xpencil", out=False); torch.cuda.synchronize()
    lib.pi_debug_xp_profile(buf)
    ctx.interact("xpencil", out=False); torch.cuda.synchronize()
    lib.pi_debug_xp_profile(buf)
    v = list(buf)
    items = 4096 * 64 // tune.get("xpencil_len", 64)
    names = ["prod wait empty", "prod fill", "prod uses", "cons wait full", "cons compute", "cons warp-uses"]
    print(tune)
    for i, n in enumerate(names):
        print(f"  {n:22s} {v[i]:16d}  per item {v[i]/items:12.0f}")
