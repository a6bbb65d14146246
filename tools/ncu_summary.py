"""Summarise an ncu report: key metrics + instruction/stall hot spots (development aid)."""
import csv, subprocess, sys
rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(det.splitlines()))
h = r[0]
want = ('Duration', 'Elapsed Cycles', 'SM Frequency', 'Executed Ipc Active', 'Issue Slots Busy', 'Achieved Occupancy',
        'Theoretical Occupancy', 'Block Limit Shared Mem', 'Block Limit Registers', 'Registers Per Thread',
        'Dynamic Shared Memory Per Block', 'Eligible Warps Per Scheduler', 'No Eligible', 'L1/TEX Cache Throughput',
        'L2 Cache Throughput', 'DRAM Throughput', 'Compute (SM) Throughput', 'Memory Throughput', 'Block Size',
        'Grid Size', 'Warp Cycles Per Issued Instruction', 'Avg. Active Threads Per Warp')
seen = set()
for row in r[1:]:
    d = dict(zip(h, row))
    k = d.get('Metric Name')
    if k in want and k not in seen:
        seen.add(k)
        print(f"{k:40s} {d['Metric Value']} {d['Metric Unit']}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(src.splitlines()))
if len(rows) > 2:
    h = rows[1]
    data = [dict(zip(h, x)) for x in rows[2:]]
    tot = sum(float(d['Instructions Executed'] or 0) for d in data)
    stot = sum(float(d['Warp Stall Sampling (All Samples)'] or 0) for d in data) or 1
    segs = []
    for d in data:
        n = float(d['Instructions Executed'] or 0); s = float(d['Warp Stall Sampling (All Samples)'] or 0)
        if segs and segs[-1][1] == n:
            segs[-1][2] += 1; segs[-1][3] += s; segs[-1][4] = d['Source'][:40]
        else:
            segs.append([d['Address'][-5:], n, 1, s, d['Source'][:40], d['Source'][:40]])
    print(f"instructions {tot:.3e}  stall samples {stot:.0f}")
    for a, n, k, s, last, first in segs:
        if n * k > 0.01 * tot or s > 0.02 * stot:
            print(f"{a} {n:10.0f} x{k:4d} = {n*k/tot*100:5.1f}%  stall {s/stot*100:5.1f}%  {first} .. {last}")
