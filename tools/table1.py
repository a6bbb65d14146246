"""The paper's Table 1 workloads on B200: uniform particles in the unit box,
d^3 cells, ppc particles per cell, the Lennard-Jones kernel (Eq. (1)), interaction kernel only,
timed like the paper (:549: 200 back-to-back calls, total / 200).  Context numbers for DESIGN.md
and BASELINE.md; bench.py is the contract.

usage: python tools/table1.py [--algos global,xpencil,fullload] [--calls 200]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_2406_16091_b200 import Context

# (d, ppc): A100 PPNL, A100 X-pencil seconds per call (BASELINE.md Table 1)
PAPER_A100 = {(8, 10): (9.1e-5, 5.6e-5), (16, 10): (1.0e-4, 8.1e-5), (32, 10): (4.2e-4, 4.0e-4),
              (8, 100): (6.1e-4, 6.1e-4), (16, 100): (3.2e-3, 3.2e-3), (32, 100): (2.5e-2, 2.5e-2)}

ap = argparse.ArgumentParser()
ap.add_argument("--algos", default="global,xpencil,fullload")
ap.add_argument("--calls", type=int, default=200)
a = ap.parse_args()
rows = []
for (d, ppc), (t_ppnl, t_xp) in PAPER_A100.items():
    n = ppc * d ** 3
    grid = synth.Grid(dims=(d, d, d), w=1.0 / d)
    c = synth.uniform(n, grid, synth.SEED_BASE + 100 + d + ppc)
    ctx = Context(grid.dims, grid.w, grid.r_c, grid.origin, kernel="lj", capacity=n,
                  lj=(grid.lj_ref, grid.lj_soft, grid.lj_e0))
    t = [torch.from_numpy(v).cuda() for v in (c.x, c.y, c.z, c.q)]
    ctx.bin(*t)
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
        paper = t_xp if algo == "xpencil" else (t_ppnl if algo == "global" else None)
        rows.append(dict(d=d, ppc=ppc, n=n, algo=algo, seconds=sec, candidates=C, rate=C / sec,
                         paper_a100_seconds=paper, speedup_vs_a100=(paper / sec if paper else None)))
        print(f"{d:3d}/{ppc:<4d} {algo:9s} {sec * 1e6:10.1f} us  {C / sec:9.3e} cand/s"
              + (f"   A100 {paper * 1e6:9.1f} us  x{paper / sec:6.1f}" if paper else ""), flush=True)
    del ctx, t
    torch.cuda.empty_cache()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(rows, open("gpurun_out/table1.json", "w"), indent=1)
