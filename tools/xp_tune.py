"""X-pencil tuning sweep on one config (development aid; bench.py is the contract).
usage: python tools/xp_tune.py CONFIG 'JSON list of {"xs": sx, tuning...}' [reps]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_16091_b200._lib as _L
if os.environ.get("LIBPI"):
    _L.LIBPATH = os.path.abspath(os.environ["LIBPI"])
import torch, synth
from paper_2406_16091_b200 import Context

cfg = sys.argv[1]
combos = json.loads(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
c = synth.make_config(cfg); g = c.grid
t = [torch.from_numpy(v).cuda() for v in (c.x, c.y, c.z, c.q)]
ci = Context(g.dims, g.w, g.r_c, g.origin, kernel="indicator", capacity=c.n)
ci.bin(t[0], t[1], t[2], torch.ones_like(t[3]))
P = float(ci.interact("global")[0].double().sum()); ci.close(); del ci
s = torch.cuda.current_stream()
for cb in combos:
    cb = dict(cb)
    xs = cb.pop("xs", 0); algo = cb.pop("algo", "xpencil")
    ctx = Context(g.dims, g.w, g.r_c, g.origin, capacity=c.n, x_subcells=xs)
    if cb: ctx.set_tuning(**cb)
    ctx.bin(*t)
    ctx.interact(algo, out=False); torch.cuda.synchronize()
    ms = []
    for r in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); ctx.interact(algo, out=False); e1.record(s); torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    ms = sorted(ms)[len(ms) // 2]
    st = ctx.stats(); C = st["candidates"]
    flop = 8 * C + 10 * P
    print(f"{cfg} {algo} xs={xs} {json.dumps(cb):40s} {ms*1e3:9.1f} us  {C/ms/1e9:6.3f} Tcand/s  "
          f"{flop/ms/1e9:6.2f} TF ({flop/ms/1e9/74.45*100:.1f}%)  fb={st['fallback_cells']}", flush=True)
    ctx.close(); del ctx
