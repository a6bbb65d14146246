"""pi_step timing with tuning variants (development aid; bench.py is the contract).
usage: python tools/step_ab.py CONFIG 'JSON list of tuning dicts' [reps]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2406_16091_b200 import Context
c = synth.make_config(sys.argv[1]); g = c.grid
combos = json.loads(sys.argv[2]); reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
t = [torch.from_numpy(v).cuda() for v in (c.x, c.y, c.z, c.q)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
for tune in combos:
    ctx = Context(g.dims, g.w, g.r_c, g.origin, capacity=c.n)
    if tune: ctx.set_tuning(**tune)
    ctx.bin(*t)
    _, fx, fy, fz = ctx.interact("xpencil")
    dt = 0.01 * g.w / float(torch.stack([fx.abs().max(), fy.abs().max(), fz.abs().max()]).max())
    ctx.bin(*t)
    for _ in range(3): ctx.step("xpencil", dt)
    ms = []
    for r in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); ctx.step("xpencil", dt); e1.record(s); torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    st = ctx.stats()
    ms = sorted(ms)[len(ms) // 2]
    print(f"{sys.argv[1]} {json.dumps(tune):28s} step {ms*1e3:9.1f} us  {st['candidates']/ms/1e9:.3f} Tcand/s  "
          f"(bin {st['bin_ms']*1e3:.0f} interact {st['interact_ms']*1e3:.0f})", flush=True)
    ctx.close(); del ctx
