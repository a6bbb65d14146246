"""Binning (a1-a4) throughput: pi_bin on random-order input and the re-binning inside pi_step
(nearly sorted input), per config.  Algorithmic bytes 48 N + 12 Nc.
Development aid; bench.py is the contract."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
from paper_2406_16091_b200 import Context

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c1,c2_ppc8,c3")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--lib", default=None, help="alternative libpi.so (A/B)")
a = ap.parse_args()
if a.lib:
    import paper_2406_16091_b200._lib as L
    L.LIBPATH = os.path.abspath(a.lib)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name in a.configs.split(","):
    c = synth.make_config(name)
    g = c.grid
    ctx = Context(g.dims, g.w, g.r_c, g.origin, capacity=c.n, device="cuda", x_subcells=int(os.environ.get("XSUB", "0")))
    t = [torch.from_numpy(v).cuda() for v in (c.x, c.y, c.z, c.q)]
    byts = 48.0 * c.n + 12.0 * g.ncells
    ms = []
    for r in range(a.reps + 2):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.bin(*t)
        e1.record()
        torch.cuda.synchronize()
        if r >= 2:
            ms.append(e0.elapsed_time(e1))
    ms_rand = sorted(ms)[len(ms) // 2]
    # re-binning inside pi_step (dt moves particles by <= 0.01 w)
    ctx.bin(*t)
    _, fx, fy, fz = ctx.interact("xpencil")
    fmax = float(torch.stack([fx.abs().max(), fy.abs().max(), fz.abs().max()]).max())
    dt = 0.01 * g.w / max(fmax, 1e-30)
    ctx.step("xpencil", dt)
    bins = []
    for r in range(a.reps + 2):
        flush.zero_()
        ctx.step("xpencil", dt)
        st = ctx.stats()
        if r >= 2:
            bins.append(st["bin_ms"])
    ms_step = sorted(bins)[len(bins) // 2]
    print(f"{name:9s} n={c.n:9d} cells={g.ncells:8d}  pi_bin (random order) {ms_rand * 1e3:8.1f} us "
          f"{byts / ms_rand / 1e6:7.0f} GB/s | pi_step re-bin {ms_step * 1e3:8.1f} us {byts / ms_step / 1e6:7.0f} GB/s")
    del ctx, t
    torch.cuda.empty_cache()
