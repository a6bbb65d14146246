"""Quick timing of the phases on one config (development aid; bench.py is the contract)."""
import argparse, json, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2406_16091_b200 import Context

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c1")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--tunes", default='[{}]')
ap.add_argument("--algos", default="global,xpencil")
a = ap.parse_args()
c = synth.make_config(a.config)
g = c.grid
dev = torch.device("cuda")
ctx = Context(g.dims, g.w, g.r_c, g.origin, capacity=c.n, device=dev)
t = [torch.from_numpy(v).to(dev) for v in (c.x, c.y, c.z, c.q)]
s = torch.cuda.current_stream()
def timeit(fn, reps):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps): fn()
    e1.record(s); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
ms_bin = timeit(lambda: ctx.bin(*t), a.reps)
ctx.bin(*t)
st = ctx.stats()
print(f"config {a.config} n={c.n} cells={g.ncells} M_C={st['max_per_cell']}")
print(f"bin: {ms_bin*1e3:.1f} us  ({(48*c.n+12*g.ncells)/ms_bin/1e6:.0f} GB/s algorithmic)")
# P (cutoff pairs) via the indicator kernel with q = 1
ci = Context(g.dims, g.w, g.r_c, g.origin, kernel="indicator", capacity=c.n, device=dev)
ci.bin(t[0], t[1], t[2], torch.ones_like(t[3]))
phi, *_ = ci.interact("global")
P = float(phi.double().sum())
for algo in a.algos.split(","):
    for tune in json.loads(a.tunes):
        if tune: ctx.set_tuning(**tune)
        ms = timeit(lambda: ctx.interact(algo, out=False), a.reps)
        st = ctx.stats()
        C = st["candidates"]
        flop = 8 * C + 10 * P
        print(f"{algo:8s} {json.dumps(tune):45s} {ms*1e3:9.1f} us  C={C:.3e} P={P:.3e} "
              f"{C/ms/1e9:8.3f} Tcand/s  {flop/ms/1e9:7.2f} TFLOP/s  ({flop/ms/1e9/74.45*100:.1f}% of 74.45)  fb={st['fallback_cells']}")
        ctx.set_tuning()
