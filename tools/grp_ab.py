"""Cell-group consumer (xpencil_targets 3 / default) vs one target per lane (1): parity on c0 (all
kernels) and c1 sampled, then timing (development aid)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from tests._util import assert_parity, gpu_interact, oracle_interact
for kernel in ["gaussian", "indicator", "lj", "lowflop", "highflop", "candidate"]:
    c = synth.make_config("c0")
    want = oracle_interact(c, kernel)
    for tpl in (1, 3):
        got, ctx = gpu_interact(c, "xpencil", kernel, tuning=dict(xpencil_targets=tpl))
        w = assert_parity(got, want, label=f"c0 {kernel} tpl{tpl}")
        print("c0", kernel, tpl, "ok worst", w, flush=True)
c = synth.make_config("c1")
sample = np.random.default_rng(2).choice(c.n, 20000, replace=False)
want = oracle_interact(c, targets=sample)
for tpl in (1, 3):
    got, ctx = gpu_interact(c, "xpencil", tuning=dict(xpencil_targets=tpl))
    print("c1", tpl, "worst", assert_parity(got[sample], want, label=f"c1 tpl{tpl}"), flush=True)
