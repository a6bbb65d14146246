"""A/B timing of pi_step and pi_interact for a given libpi build (development aid).
usage: python tools/ab.py LIBPATH [config] [algo]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_16091_b200._lib as L
L.LIBPATH = os.path.abspath(sys.argv[1])
import torch, synth
from paper_2406_16091_b200 import Context
cfg = sys.argv[2] if len(sys.argv) > 2 else "c1"
algo = sys.argv[3] if len(sys.argv) > 3 else "xpencil"
c = synth.make_config(cfg); g = c.grid
ctx = Context(g.dims, g.w, g.r_c, g.origin, capacity=c.n, x_subcells=int(os.environ.get('XSUB', '0')))
if any(os.environ.get(k) for k in ("TPL", "LEN", "TGT", "THREADS", "CAP")):
    ctx.set_tuning(xpencil_slots=int(os.environ.get('TPL', '0')), threads=int(os.environ.get('THREADS', '0')),
                   xpencil_len=int(os.environ.get('LEN', '0')), xpencil_targets=int(os.environ.get('TGT', '0')),
                   xpencil_cap=int(os.environ.get('CAP', '0')))
t = [torch.from_numpy(v).cuda() for v in (c.x, c.y, c.z, c.q)]
ctx.bin(*t)
_, fx, fy, fz = ctx.interact(algo)
dt = 0.01 * g.w / float(torch.stack([fx.abs().max(), fy.abs().max(), fz.abs().max()]).max())
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def run(fn, reps=20):
    ms = []
    for r in range(reps + 3):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        if r >= 3: ms.append(e0.elapsed_time(e1))
    return sorted(ms)[len(ms) // 2]
ctx.bin(*t)
ctx.step(algo, dt)
step = run(lambda: ctx.step(algo, dt))
st = ctx.stats()
ctx.bin(*t)
inter = run(lambda: ctx.interact(algo, out=False))
print(f"{os.path.basename(L.LIBPATH):20s} slots={os.environ.get('TPL', '0')} len={os.environ.get('LEN', '0')} thr={os.environ.get('THREADS', '0')} tgt={os.environ.get('TGT', '0')} cap={os.environ.get('CAP', '0')} sx={os.environ.get('XSUB', '0')} {cfg} {algo}: step {step*1e3:7.1f} us (bin {st['bin_ms']*1e3:6.1f} interact {st['interact_ms']*1e3:6.1f})  pi_interact {inter*1e3:7.1f} us")
