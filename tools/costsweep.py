"""Kernel-cost sweep (the paper's Fig. "diffflops" experiment): one workload,
every interaction strategy, kernels from cheap to costly -- CANDIDATE (count every 27-cell
candidate: no distance), INDICATOR (distance + cutoff test), the paper's 5-FLOP fake kernel
LOWFLOP ("summing the positions"), Gaussian (+ ex2), Lennard-Jones (Eq. (1), the paper's 18-21
FLOP kernel) and the paper's 168-FLOP fake kernel HIGHFLOP (LJ + 150 FLOP; reading R22).
Interaction kernel only, 200 back-to-back calls as PAPER.md:549.
Context for DESIGN.md; bench.py is the contract.

usage: python tools/costsweep.py [--config c1] [--calls 200]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
from paper_2406_16091_b200 import Context

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c1")
ap.add_argument("--calls", type=int, default=200)
ap.add_argument("--algos", default="global,fullload,xpencil")
a = ap.parse_args()
c = synth.make_config(a.config)
g = c.grid
t = [torch.from_numpy(v).cuda() for v in (c.x, c.y, c.z, c.q)]
rows = []
for kernel in ("candidate", "indicator", "lowflop", "gaussian", "lj", "highflop"):
    ctx = Context(g.dims, g.w, g.r_c, g.origin, kernel=kernel, capacity=c.n,
                  lj=(g.lj_ref, g.lj_soft, g.lj_e0) if kernel in ("lj", "highflop") else (0, 0, 0))
    ctx.bin(*t)
    line = f"{kernel:10s}"
    for algo in a.algos.split(","):
        ctx.interact(algo, out=False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.calls):
            ctx.interact(algo, out=False)
        e1.record()
        torch.cuda.synchronize()
        sec = e0.elapsed_time(e1) / 1e3 / a.calls
        C = ctx.stats()["candidates"]
        rows.append(dict(config=a.config, kernel=kernel, algo=algo, seconds=sec, candidates=C, rate=C / sec))
        line += f"  {algo} {sec * 1e6:8.1f} us ({C / sec:.3e} cand/s)"
    print(line, flush=True)
    ctx.close()
    del ctx
os.makedirs("gpurun_out", exist_ok=True)
json.dump(rows, open(f"gpurun_out/costsweep_{a.config}.json", "w"), indent=1)
