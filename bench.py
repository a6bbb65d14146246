#!/usr/bin/env python
"""bench.py -- throughput of the hot path of arXiv 2406.16091 on B200 (driver contract).

A "step" is one pass of the whole hot path over the synthetic cloud of BASELINE.json
configs[4] (2^27 uniform particles, 256^3 cells, 8 per cell, Gaussian K, r_c = w -- the
configuration the metric "pair interactions/s and step ms at 1/2/4/8 B200" is quoted on):
pi_step = a1-a4 binning (cell index + counts, scan + M_C, scatter), a5-a6 interaction
(X-pencil strategy by default) and a7 position update.  Inputs are resident in HBM (2 GiB of
records: larger than L2, and L2 is flushed with a 256 MiB write between timed steps, outside
the timed events).  The metric is candidate pair interactions per second (ordered pairs (i, j),
j != i, in the 27 neighbour cells -- the unit of the paper's Table 1).
configs[1] (2^21, 64^3; round 1's workload) is reported beside it under "config_c1".

  python bench.py [--gpus N] [--steps K] [--warmup W] [--algo xpencil|global|fullload]
                  [--scaling strong|weak] [--config c4|c1|...]
  python bench.py --impl reference ...   # the fp64 CPU oracle on a bounded sample (rank 0)

N > 1 (launched with torchrun): the X-slab decomposition (a8); each pi_step
migrates particles and exchanges ghost layers with the X neighbours over NCCL.
  --scaling strong (default): configs[4] itself, 2^27 particles on 256^3 cells split into
      N X-slabs of 256/N layers ("scaling": "strong").
  --scaling weak: 2^24 particles per GPU on a (32 N) x 256 x 256 grid (equal to
      configs[4] at N = 8) ("scaling": "weak").
Timed on the device, MAX over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP32_PEAK_TFLOPS = 2 * 128 * 148 * 1.965e9 / 1e12  # 74.45: FMA lanes x SMs x max SM clock
METRIC = "candidate pair interactions/s (27-cell ordered pairs), step ms"
WORKLOADS = {
    "c4": ("BASELINE configs[4]: 2^27 uniform particles in the unit box, 256^3 cells (8/cell), "
           "r_c = w = 1/256, Gaussian K sigma = r_c/3, fp32, one B200"),
    "c1": ("BASELINE configs[1]: 2^21 uniform particles in the unit box, 64^3 cells (8/cell), "
           "r_c = w = 1/64, Gaussian K sigma = r_c/3, fp32"),
}


def fp32_peak_measured():
    """The FFMA2 peak measured by tools/pipes.cu on a B200 of this pool (profiles/peaks.json)."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "peaks.json")))
        return float(d["ffma2_tflops"]), d.get("how", "tools/pipes.cu")
    except Exception:
        return None, None


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--no-c1", action="store_true", help="skip the configs[1] side measurement")
    ap.add_argument("--algo", default="xpencil")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-binning-2e24", action="store_true", help="skip the 2^24 binning measurement")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------------------ clocks
class ClockSampler:
    """NVML samples of SM clock and throttle reasons while the timed region runs."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = set()
        self._stop = threading.Event()
        self._t = None
        self.max_mhz = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._nv = pynvml
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception:
            self._nv = None
        return self

    def _run(self):
        nv = self._nv
        names = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                 "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.005)

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ------------------------------------------------------------------------ helpers
def traffic_from_profiles(algo):
    """dram read+write bytes per launch of the interaction kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        return json.load(open(p)).get(algo)
    except Exception:
        return None


def smem_from_profiles(algo):
    """Shared-memory wavefronts of the interaction kernel as a fraction of their peak, from the
    committed ncu capture (the X-pencil's binding resource), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_smem.json")
    try:
        return json.load(open(p)).get(algo)
    except Exception:
        return None


def oracle_subcloud(cloud, max_n=1 << 22):
    """A bounded sample of the workload for the CPU oracle: the particles of the first X layers of
    the grid (whole layers, same cells, density and kernel), about max_n of them, so the oracle's
    own binning of the sample stays bounded (binning all 2^27 particles of configs[4] takes it ~6 s
    single-threaded).  Returns (sub-cloud, description)."""
    import numpy as np
    import synth
    g = cloud.grid
    if cloud.n <= max_n:
        return cloud, f"the whole {cloud.n}-particle cloud"
    lx = max(1, int(round(g.dims[0] * max_n / cloud.n)))
    xmax = np.float32(g.origin[0] + lx * g.w)
    m = cloud.x < xmax
    sub = synth.Cloud(synth.Grid(dims=(lx, g.dims[1], g.dims[2]), w=g.w, origin=g.origin, rc=g.rc, sigma=g.sigma),
                      cloud.x[m], cloud.y[m], cloud.z[m], cloud.q[m], name=f"{cloud.name}-x{lx}")
    return sub, f"the {sub.n} particles of the first {lx} X layers ({lx}x{g.dims[1]}x{g.dims[2]} cells) of the cloud"


def oracle_rate(cloud, seconds, threads, rng_seed=7):
    """The fp64 cell-list oracle as it stands, on a bounded random sample of targets."""
    import numpy as np
    from oracle import celllist
    celllist.set_threads(threads)
    rng = np.random.default_rng(rng_seed)
    probe = rng.choice(cloud.n, min(cloud.n, 20000), replace=False)
    t0 = time.perf_counter()
    r = celllist.interact(cloud.x, cloud.y, cloud.z, cloud.q, cloud.grid, targets=probe)
    dt = time.perf_counter() - t0
    per_target = dt / len(probe)
    m = int(min(cloud.n, max(len(probe), seconds / max(per_target, 1e-9))))
    sample = rng.choice(cloud.n, m, replace=False)
    t0 = time.perf_counter()
    r = celllist.interact(cloud.x, cloud.y, cloud.z, cloud.q, cloud.grid, targets=sample)
    dt = time.perf_counter() - t0
    cands = int(r["C"].sum())
    return cands / dt, dict(targets=m, candidates=cands, seconds=dt)


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ------------------------------------------------------------------------ workload (both arms)
def workload_cloud(a, rank, world):
    """This rank's synthetic input: configs[4] (or --config) at N = 1; at N > 1 this rank's X-slab
    of configs[4] (strong) or of the (32 N) x 256 x 256 weak-scaling grid."""
    import synth
    if world > 1 or a.scaling == "weak":
        lx = 32 if a.scaling == "weak" else 256 // world
        # uniform inside the rank's slab, 8 per cell, w = 1/256 (an independent stream per rank: the
        # union is a uniform cloud of the same statistics as synth.make_config("c4"))
        return synth.slab_uniform(8.0, (lx, 256, 256), rank, world, seed=synth.SEED_BASE + 4)
    return synth.make_config(a.config)


def workload_config(a, world, cloud, n_total):
    g = cloud.grid
    if world > 1 or a.scaling == "weak":
        if a.scaling == "weak":
            workload = (f"configs[4] weak scaling (SURVEY.md Q22): {g.dims[0]}x{g.dims[1]}x{g.dims[2]} cells, 32 X "
                        "layers (2^24 uniform particles, 8 per cell) per GPU, r_c = w = 1/256, Gaussian K sigma = r_c/3, "
                        "fp32; NCCL ghost + migration exchange every step")
        else:
            workload = (f"BASELINE configs[4] strong scaling: 2^27 uniform particles, 256^3 cells (8/cell) in {world} "
                        f"X-slabs of {g.dims[0] // world} layers, r_c = w = 1/256, Gaussian K sigma = r_c/3, fp32; NCCL "
                        "ghost + migration exchange every step")
    elif a.config in WORKLOADS:
        workload = WORKLOADS[a.config]
    else:
        workload = f"synth.make_config({a.config!r}): {cloud.n} particles, {tuple(g.dims)} cells, Gaussian K, fp32"
    return {"workload": workload, "n_per_gpu": cloud.n, "n_total": int(n_total), "cells": g.ncells,
            "algo": a.algo, "step": "pi_step: re-bin (scan of the carried counts + scatter) + interact + integrate"
            + (" + a8 migration/ghost exchange (NCCL)" if world > 1 else ""),
            "l2": "inputs larger than L2 (2 GiB of records at configs[4]) and L2 flushed between timed steps "
                  "(256 MiB write, outside the events)",
            "parallelism": f"xslab{world}" if world > 1 else "single GPU"}


def scaling_of(a, world):
    return a.scaling


# ------------------------------------------------------------------------ reference arm
def run_reference(a):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cloud = workload_cloud(a, 0, world)
    sub, desc = oracle_subcloud(cloud)
    cores = host_cores()
    per_step = max(1.0, min(10.0, 120.0 / max(1, a.steps + a.warmup)))
    rates = []
    info = None
    for s in range(a.warmup + a.steps):
        rate, info = oracle_rate(sub, per_step, cores, rng_seed=100 + s)
        if s >= a.warmup:
            rates.append(rate)
    value = statistics.mean(rates)
    unit = "candidate pair interactions/s"
    ms = info["seconds"] * 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": value,
        "unit": unit, "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": scaling_of(a, world), "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": workload_config(a, world, cloud, cloud.n * world),
        "cpu_baseline": {"value": value, "unit": unit, "cores": cores, "kind": "oracle",
                         "sample": f"{info['targets']} random targets of {desc} per step "
                                   f"(fp64 C cell list, OpenMP, {cores} threads; includes its own binning of the sample)"},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------ binning at 2^24
def binning_at_scale(a, dev, stream, flush):
    """The binning phase's HBM roofline at 2^24 particles, 128^3 cells (configs[2] ppc 8; configs[1]
    is L2-resident): the pi_step re-binning (the method's steady state, nearly sorted input) and
    the first pi_bin of random-order input, device time from the library's phase events."""
    import statistics as st
    import torch
    import synth
    from paper_2406_16091_b200 import Context
    c = synth.make_config("c2_ppc8")
    g = c.grid
    ctx = Context(g.dims, g.w, g.r_c, g.origin, capacity=c.n, device=dev, stream=stream)
    x, y, z, q = (torch.from_numpy(v).to(dev) for v in (c.x, c.y, c.z, c.q))
    first = []
    for _ in range(3):
        flush.zero_()
        ctx.bin(x, y, z, q)
        first.append(ctx.stats()["bin_ms"])
    _, fx, fy, fz = ctx.interact(a.algo)
    fm = float(torch.stack([fx.abs().max(), fy.abs().max(), fz.abs().max()]).max())
    dt = 0.01 * g.w / max(fm, 1e-30)
    del fx, fy, fz
    ctx.step(a.algo, dt)
    rebin = []
    for _ in range(8):
        flush.zero_()
        ctx.step(a.algo, dt)
        rebin.append(ctx.stats()["bin_ms"])
    ctx.close()
    byts = 48.0 * c.n + 12.0 * g.ncells
    peak = hbm_peak_gbs()
    r_ms, f_ms = st.median(rebin), st.median(first)
    return {"workload": "2^24 uniform particles, 128^3 cells (configs[2] ppc 8)", "bytes_model": "48 B/particle + 12 B/cell",
            "rebin_ms": r_ms, "rebin_gbs": byts / (r_ms * 1e-3) / 1e9, "rebin_frac": byts / (r_ms * 1e-3) / 1e9 / peak,
            "first_bin_ms": f_ms, "first_bin_gbs": byts / (f_ms * 1e-3) / 1e9,
            "first_bin_frac": byts / (f_ms * 1e-3) / 1e9 / peak, "peak_gbs": peak,
            "peak_basis": "MEASURED_PEAKS.json hbm_gbs (copy)"}


def side_config(a, dev, stream, flush, name):
    """pi_step of another BASELINE config (device time per step and candidate pairs/s), for
    continuity with earlier rounds (configs[1] was round 1's bench workload)."""
    import torch
    import synth
    from paper_2406_16091_b200 import Context
    c = synth.make_config(name)
    g = c.grid
    ctx = Context(g.dims, g.w, g.r_c, g.origin, capacity=c.n, device=dev, stream=stream)
    x, y, z, q = (torch.from_numpy(v).to(dev) for v in (c.x, c.y, c.z, c.q))
    ctx.bin(x, y, z, q)
    _, fx, fy, fz = ctx.interact(a.algo)
    dt = 0.01 * g.w / max(float(torch.stack([fx.abs().max(), fy.abs().max(), fz.abs().max()]).max()), 1e-30)
    del fx, fy, fz
    for _ in range(3):
        ctx.step(a.algo, dt)
    ms, ims, cs = [], [], []
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ctx.step(a.algo, dt)
        e1.record(stream)
        st = ctx.stats()
        ms.append(e0.elapsed_time(e1))
        ims.append(st["interact_ms"])
        cs.append(st["candidates"])
    ctx.close()
    m = statistics.median(ms)
    return {"workload": WORKLOADS.get(name, name), "ms_per_step": m, "value": statistics.mean(cs) / (m * 1e-3),
            "interact_ms": statistics.median(ims), "unit": "candidate pair interactions/s"}


def strategies_at(a, dev, stream, name="c1"):
    """pi_interact of every strategy on one config (device time, candidate pairs/s): the paper's
    strategy comparison (Table 1 / Fig. perf) incl. X-pencil-reg (NEXT #1)."""
    import torch
    import synth
    from paper_2406_16091_b200 import Context
    c = synth.make_config(name)
    g = c.grid
    ctx = Context(g.dims, g.w, g.r_c, g.origin, capacity=c.n, device=dev, stream=stream)
    x, y, z, q = (torch.from_numpy(v).to(dev) for v in (c.x, c.y, c.z, c.q))
    ctx.bin(x, y, z, q)
    out = {"workload": WORKLOADS.get(name, name), "unit": "candidate pair interactions/s"}
    for algo in ("global", "fullload", "xpencil", "xpreg", "half"):
        ctx.interact(algo, out=False)
        ms = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ctx.interact(algo, out=False)
            e1.record(stream)
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
        m = statistics.median(ms)
        out[algo] = {"interact_ms": m, "value": ctx.stats()["candidates"] / (m * 1e-3)}
    ctx.close()
    return out


def hbm_peak_gbs():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0  # B200_PROFILING.md fallback


# ------------------------------------------------------------------------ our arm
def run_ours(a):
    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    from paper_2406_16091_b200 import Context, nccl_unique_id

    rank, world, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", init_method="env://")
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)
    cloud = workload_cloud(a, rank, world)
    g = cloud.grid
    n = cloud.n
    cap = int(n * 1.25) + 4096 if world > 1 else n  # owned + ghosts + migration slack
    stream = torch.cuda.current_stream(dev)

    def make_ctx(kernel="gaussian"):
        kw = {}
        if world > 1:
            obj = [nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            kw = dict(rank=rank, nranks=world, nccl_unique_id=obj[0])
        return Context(g.dims, g.w, g.r_c, g.origin, kernel=kernel, capacity=cap, device=dev, stream=stream, **kw)

    ctx = make_ctx()
    x, y, z, q = (torch.from_numpy(v).to(dev) for v in (cloud.x, cloud.y, cloud.z, cloud.q))

    # cutoff pairs P of this rank's targets (pi_count_pairs: the global baseline's walk over the
    # sorted state) for the algorithmic FLOP count 8 C + 10 P of this rank's interaction kernel
    ctx.bin(x, y, z, q)
    P = float(ctx.count_pairs())

    # dt: max |dt F| <= 0.01 w, the same on every rank
    ctx.bin(x, y, z, q)
    _, fx, fy, fz = ctx.interact(a.algo)
    fm = torch.stack([fx.abs().max(), fy.abs().max(), fz.abs().max()]).max().double().reshape(1)
    if world > 1:
        dist.all_reduce(fm, op=dist.ReduceOp.MAX)
    dt = 0.01 * g.w / max(float(fm.item()), 1e-30)
    del fx, fy, fz

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(a.steps)]
    ctx.bin(x, y, z, q)
    clk = ClockSampler(dev.index or 0).__enter__()   # samples from warm-up to the end of e2e
    for _ in range(a.warmup):
        ctx.step(a.algo, dt)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    inter_ms, bin_ms, exch_ms, cands, migr = [], [], [], [], []
    for k in range(a.steps):
        flush.zero_()                      # evict L2 (outside the timed events)
        ev[k][0].record(stream)
        ctx.step(a.algo, dt)
        ev[k][1].record(stream)
        st = ctx.stats()                   # synchronises; per-phase device times of this step
        inter_ms.append(st["interact_ms"])
        bin_ms.append(st["bin_ms"])
        exch_ms.append(st["exchange_ms"])
        cands.append(st["candidates"])
        migr.append(st["migrants_in"])
    torch.cuda.synchronize()
    step_ms = [e0.elapsed_time(e1) for e0, e1 in ev]
    if world > 1:
        dist.barrier()
    tot_ms = sum(step_ms)
    tot_c = float(sum(cands))
    n_all = float(n)
    if world > 1:
        t = torch.tensor([tot_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
        c = torch.tensor([tot_c, n_all], device=dev, dtype=torch.float64)
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
        tot_c, n_all = float(c[0].item()), float(c[1].item())
    value = tot_c / (tot_ms * 1e-3)
    C = statistics.mean(cands)
    flop = 8.0 * C + 10.0 * P
    int_ms = statistics.mean(inter_ms)
    achieved = flop / (int_ms * 1e-3) / 1e12
    pk_meas, _ = fp32_peak_measured()
    bin_bytes = 48.0 * n + 12.0 * g.ncells / world

    # end to end through the C ABI on pinned host buffers (H2D + bin (+ a8) + interact + D2H).
    # One rank: pi_run_host_submit/_wait, three runs in flight (run k+1's upload and run k-1's
    # download overlap run k's kernels); every run still copies its own inputs up and its
    # outputs down inside the timed region.  Also timed: the synchronous pi_run_host.
    hx, hy, hz, hq = (torch.from_numpy(v).pin_memory() for v in (cloud.x, cloud.y, cloud.z, cloud.q))
    ho = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(4)]
    for _ in range(2):
        ctx.run_host(a.algo, hx, hy, hz, hq, *ho)
    e2e_sync = []
    for _ in range(max(3, min(a.steps // 2, 6))):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ctx.run_host(a.algo, hx, hy, hz, hq, *ho)
        e1.record(stream)
        e1.synchronize()
        e2e_sync.append(e0.elapsed_time(e1))
    e2e_sync_ms = statistics.mean(e2e_sync)
    if world == 1:
        ho2 = [ho] + [[torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(4)] for _ in range(2)]
        runs = max(6, min(a.steps, 12))
        for k in range(4):
            ctx.run_host_submit(a.algo, hx, hy, hz, hq, *ho2[k % 3])
        ctx.run_host_wait()
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for k in range(runs):
            ctx.run_host_submit(a.algo, hx, hy, hz, hq, *ho2[k % 3])
        ctx.run_host_wait()
        e1.record(stream)
        e1.synchronize()
        e2e_ms = [e0.elapsed_time(e1) / runs]
        e2e_path = ("pi_run_host_submit/_wait, 3 runs in flight: pinned H2D x,y,z,q -> bin -> interact -> "
                    "D2H phi,F per run, copies overlapping the previous/next run's kernels")
        # the host link's floor for this run: the same bytes up and down at once, plain copies
        dev_in = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(4)]
        dev_out = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(4)]
        su, sd = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        def both():
            with torch.cuda.stream(su):
                for d_, h_ in zip(dev_in, (hx, hy, hz, hq)):
                    d_.copy_(h_, non_blocking=True)
            with torch.cuda.stream(sd):
                for h_, d_ in zip(ho, dev_out):
                    h_.copy_(d_, non_blocking=True)
        both()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        su.wait_stream(stream)
        sd.wait_stream(stream)
        for _ in range(5):
            both()
        stream.wait_stream(su)
        stream.wait_stream(sd)
        e1.record(stream)
        e1.synchronize()
        link_floor_ms = e0.elapsed_time(e1) / 5
        del dev_in, dev_out
    else:
        link_floor_ms = None
        e2e_ms = e2e_sync
        e2e_path = "pi_run_host: pinned H2D x,y,z,q -> bin -> a8 exchange -> interact -> D2H phi,F"
    c_e2e = float(ctx.stats()["candidates"])
    clk.__exit__()
    e2e_mean = statistics.mean(e2e_ms)
    if world > 1:
        t = torch.tensor([e2e_mean], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_mean = float(t.item())
        c = torch.tensor([c_e2e], device=dev, dtype=torch.float64)
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
        c_e2e = float(c.item())
    e2e_value = c_e2e / (e2e_mean * 1e-3)

    if world > 1 and a.algo == "xpencil" and g.dims[0] // world >= 4:
        # the overlapped step: stayers, append migrants, append ghosts, count,
        # scan, scatter (which writes the source pairs); the boundary and the interior X-pencil
        # launches, each with its Par-Cell-SM kernel; on the exchange stream 2 header resets, the
        # boundary sort and the arrivals' ghost selection; NCCL's own kernels not counted
        launches = 14
    elif world > 1:
        # reset, migrate, append, reset, ghosts, append, count, scan, scatter (which writes the
        # source pairs), interact (+ the Par-Cell-SM kernel of the full load and the X-pencil);
        # NCCL's own kernels not counted
        launches = 10 + (1 if a.algo in ("fullload", "xpencil") else 0)
    else:
        # pi_step, one rank: scan of the carried counts (k_scan_delta), scatter (which also
        # writes the X-pencil's source pairs), interact (+ integrate fused); plus two memsets of
        # the control block, not counted.  The full load and the X-pencil add their Par-Cell-SM
        # kernel (the cells listed for it that no block took during the interaction kernel).
        launches = 3 + (1 if a.algo in ("fullload", "xpencil") else 0)
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "candidate pair interactions/s",
        "n_gpus": world,
        "steps": a.steps,
        "warmup": a.warmup,
        "ms_per_step": tot_ms / a.steps,
        "higher_is_better": True,
        "scaling": scaling_of(a, world),
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic",
        "config": workload_config(a, world, cloud, n_all),
        "roofline": {"bound": "alu", "achieved": achieved, "peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": achieved / FP32_PEAK_TFLOPS, "traffic": traffic_from_profiles(a.algo),
                     "smem_wavefront_frac_ncu": smem_from_profiles(a.algo),
                     "kernel": f"k_interact_{a.algo}", "flop_per_launch": flop,
                     "flop_model": "8 per candidate + 10 per cutoff pair (SURVEY.md §8(d))",
                     "candidates": C, "cutoff_pairs": P, "kernel_ms": int_ms,
                     "peak_basis": "nominal 2 x 128 FP32 lanes x 148 SMs x 1.965 GHz (MEASURED_PEAKS.json has no "
                                   "FP32 entry); frac_measured: against the FFMA2 rate measured by tools/pipes.cu "
                                   "(profiles/peaks.json)",
                     "peak_measured": pk_meas,
                     "frac_measured": (achieved / pk_meas) if pk_meas else None,
                     "note": ("effective rate: the unit is the 27-cell candidate pair, but the X-pencil skips "
                              "the X sub-cells farther than r_c from the target (exact; DESIGN.md R18)"
                              if a.algo == "xpencil" else "every 27-cell candidate is evaluated")},
        "phases": {"bin_ms": statistics.mean(bin_ms), "interact_ms": int_ms,
                   "exchange_ms": statistics.mean(exch_ms) if world > 1 else 0.0,
                   "migrants_per_step": statistics.mean(migr) if world > 1 else 0.0,
                   "bin_gbs_algorithmic": bin_bytes / (statistics.mean(bin_ms) * 1e-3) / 1e9,
                   "bin_bytes_model": "48 B/particle + 12 B/cell"},
        "e2e": {"value": e2e_value, "unit": "candidate pair interactions/s", "ms": e2e_mean,
                "h2d_bytes_per_step": 16 * n, "d2h_bytes_per_step": 16 * n,
                "path": e2e_path, "sync_ms": e2e_sync_ms,
                "link_floor_ms": link_floor_ms,
                "link_note": "the same H2D + D2H bytes copied at once with plain copies (the host link's floor)"},
        "gpu_launches": launches * a.steps,
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cores = host_cores()
        sub, desc = oracle_subcloud(cloud)
        rate, info = oracle_rate(sub, a.cpu_seconds, cores)
        line["cpu_baseline"] = {"value": rate, "unit": "candidate pair interactions/s", "cores": cores,
                                "kind": "oracle",
                                "sample": f"{info['targets']} random targets of {desc} "
                                          f"({info['candidates']} candidates, {info['seconds']:.1f} s, fp64 C "
                                          "cell list incl. its own binning of the sample)"}
    if world == 1 and not a.no_binning_2e24:
        line["binning_2e24"] = binning_at_scale(a, dev, stream, flush)
    if world == 1 and not a.no_c1 and a.config != "c1":
        line["config_c1"] = side_config(a, dev, stream, flush, "c1")
    if world == 1 and not a.no_c1:
        line["strategies_c1"] = strategies_at(a, dev, stream, "c1")
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
