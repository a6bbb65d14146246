"""Builds profiles/<round>_ncu_summary.md, profiles/ncu_traffic.json and ncu_smem.json from the ncu reports
of tools/profile_round.sh (gpurun_out/<round>_*).  Development aid."""
import csv, json, os, subprocess, sys
from collections import defaultdict

R = sys.argv[1] if len(sys.argv) > 1 else "r01"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__cycles_elapsed.avg.per_second",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "smsp__inst_executed.sum",
        "sm__inst_executed.avg.per_cycle_active", "launch__grid_size", "launch__block_size",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]


SCALE = {"ns": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "s": 1e9, "second": 1e9, "nsecond": 1.0,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "hz": 1.0, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "cycle/second": 1.0, "cycle/nsecond": 1e9,
         "cycle/usecond": 1e6, "cycle/msecond": 1e3}


def raw(rep):
    """Rows of the raw page with values normalised to ns / bytes / Hz."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for k, u, v in zip(h, units, r):
            if k in KEYS:
                try:
                    x = float(v.replace(",", ""))
                    d[k] = str(x * SCALE.get(u, 1.0))
                except ValueError:
                    d[k] = v
            else:
                d[k] = v
        res.append(d)
    return res


def fmt(d):
    t = float(d["gpu__time_duration.sum"]) / 1e3  # ns -> us
    rd, wr = float(d["dram__bytes_read.sum"]), float(d["dram__bytes_write.sum"])
    f = float(d.get("sm__cycles_elapsed.avg.per_second", 0) or 0) / 1e9
    return (f"- duration {t:.1f} us at {f:.3f} GHz; DRAM read {rd / 1e6:.2f} MB + write {wr / 1e6:.2f} MB "
            f"= {(rd + wr) / 1e6:.2f} MB ({(rd + wr) / (t * 1e-6) / 1e9:.0f} GB/s)\n"
            f"- FMA pipe active {float(d['sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active']):.1f} %, "
            f"FMA-pipe instructions {float(d['sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active']):.1f} % of peak, "
            f"XU (MUFU) {float(d['sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active']):.1f} %, "
            f"warps active {float(d['sm__warps_active.avg.pct_of_peak_sustained_active']):.1f} %, "
            f"IPC {float(d['sm__inst_executed.avg.per_cycle_active']):.2f}, "
            f"registers {d['launch__registers_per_thread']}, grid {d['launch__grid_size']} x {d['launch__block_size']}, "
            f"warp instructions {int(float(d['smsp__inst_executed.sum'])):,}"), rd + wr


out = [f"# {R}: ncu summaries (B200, `--set full --clock-control none`, one capture per kernel)\n",
       "Captured by `tools/profile_round.sh` under gpurun; raw reports stay in gpurun_out/ (not tracked).",
       "Durations under ncu are serialised and cold-cache: compare shares, not absolute times (bench.py",
       "times the kernels live with CUDA events).\n"]
traffic, smem = {}, {}
for name, title in (("xpencil_c4", "X-pencil interaction, the bench kernel (configs[4], 2^27, 256^3)"),
                    ("xpencil", "X-pencil interaction (configs[1], 2^21, 64^3)"),
                    ("global", "global-memory baseline PPNL (configs[1])"),
                    ("fullload", "full-load interaction (configs[1])"),
                    ("xpreg", "X-pencil-reg interaction (configs[1])")):
    rep = os.path.join(G, f"{R}_{name}.ncu-rep")
    if not os.path.exists(rep):
        continue
    for d in raw(rep):
        s, tr = fmt(d)
        out.append(f"## {title}: `{d['Kernel Name'][:60]}`\n{s}\n")
        key = "xpencil" if name == "xpencil_c4" else (name + "_c1" if name == "xpencil" else name)
        traffic[key] = int(tr)
        w = d.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed")
        if w not in (None, ""):
            smem[key] = round(float(w) / 100.0, 4)
for name, title in (("rebin", "binning, pi_step delta re-binning on configs[4] (2^27: scan of the carried counts + scatter of the nearly sorted records)"),
                    ("bin", "binning, pi_bin at 2^24 (configs[2] ppc 8, random input order)")):
    rep = os.path.join(G, f"{R}_{name}.ncu-rep")
    if not os.path.exists(rep):
        continue
    out.append(f"## {title}\n")
    for d in raw(rep):
        s, _ = fmt(d)
        out.append(f"### `{d['Kernel Name'][:70]}`\n{s}\n")
# launch list shares
ll = os.path.join(G, f"{R}_launches.csv")
if os.path.exists(ll):
    rows = [r for r in csv.reader(open(ll)) if len(r) > 10]
    h = rows[0]
    iK, iV = h.index("Kernel Name"), h.index("Metric Value")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        k = r[iK].split("(")[0].replace("void ", "").replace("unnamed>::", "")
        tot[k] += float(r[iV])
        cnt[k] += 1
    s = sum(tot.values())
    out.append("## Launch list of `bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-binning-2e24 --no-c1` "
               "(configs[4]; all kernels of the run, ncu-serialised)\n")
    out.append("| kernel | launches | total us | share |\n|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        out.append(f"| `{k}` | {cnt[k]} | {v / 1e3:.1f} | {100 * v / s:.1f} % |")
open(os.path.join(ROOT, "profiles", f"{R}_ncu_summary.md"), "w").write("\n".join(out) + "\n")
json.dump(traffic, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
json.dump(smem, open(os.path.join(ROOT, "profiles", "ncu_smem.json"), "w"), indent=1)
print("\n".join(out))
print(traffic)
