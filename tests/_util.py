"""Helpers shared by the GPU parity tests (CUDA path through the C ABI vs the oracle)."""
from __future__ import annotations

import numpy as np
import torch

from oracle import celllist
from oracle import reference as ref


def ctx_for(cloud, kernel="gaussian", capacity=None, **kw):
    from paper_2406_16091_b200 import Context
    g = cloud.grid
    cap = capacity if capacity is not None else max(cloud.n, 1)
    if kernel in ("lj", "highflop"):
        kw.setdefault("lj", (g.lj_ref, g.lj_soft, g.lj_e0))
    return Context(g.dims, g.w, g.r_c, g.origin, kernel=kernel, sigma=0.0 if g.sigma is None else g.sigma,
                   capacity=cap, device="cuda", **kw)


def to_dev(cloud):
    # torch allocations are 512-B aligned, as the ABI requires (16 B)
    return [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (cloud.x, cloud.y, cloud.z, cloud.q)]


def gpu_interact(cloud, algo, kernel="gaussian", tuning=None, ctx=None):
    if ctx is None:
        ctx = ctx_for(cloud, kernel)
    if tuning:
        ctx.set_tuning(**tuning)
    ctx.bin(*to_dev(cloud))
    phi, fx, fy, fz = ctx.interact(algo)
    torch.cuda.synchronize()
    out = torch.stack([phi, fx, fy, fz], 1).cpu().numpy().astype(np.float64)
    return out, ctx


KERNEL_ID = {"gaussian": ref.KERNEL_GAUSSIAN, "indicator": ref.KERNEL_INDICATOR, "candidate": ref.KERNEL_CANDIDATE,
             "lj": ref.KERNEL_LJ, "lowflop": ref.KERNEL_LOWFLOP, "highflop": ref.KERNEL_HIGHFLOP}


def oracle_interact(cloud, kernel="gaussian", targets=None, band=None):
    return celllist.interact(cloud.x, cloud.y, cloud.z, cloud.q, cloud.grid, kernel=KERNEL_ID[kernel],
                             targets=targets, band=band)


def assert_parity(got, want, rel=1e-4, label=""):
    ok, worst, where = ref.check_interactions(got, want, rel=rel)
    if not ok:
        i = where[0] if where is not None else None
        detail = ""
        if i is not None:
            detail = f" row {i}: gpu {got[i]} oracle {want['out'][i]} S {want['S'][i]} A {want['A'][i]}"
        raise AssertionError(f"{label}: parity failed, worst err/bound = {worst:.3g}{detail}")
    return worst
