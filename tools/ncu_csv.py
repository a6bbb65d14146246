"""Summarise exported ncu pages (tools/ncu_export.sh): key metrics and per-basic-block instruction
shares.  usage: python tools/ncu_csv.py PREFIX [min_share]   (PREFIX.details.csv, PREFIX.source.csv.gz)"""
import csv, gzip, io, sys
pre = sys.argv[1]
mn = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
rows = list(csv.reader(open(pre + ".details.csv")))
h = rows[0]
want = ('Duration', 'Executed Ipc Active', 'Issue Slots Busy', 'Achieved Occupancy', 'Registers Per Thread',
        'Eligible Warps Per Scheduler', 'No Eligible', 'L1/TEX Cache Throughput', 'DRAM Throughput',
        'Compute (SM) Throughput', 'Warp Cycles Per Issued Instruction', 'Avg. Active Threads Per Warp',
        'Executed Instructions', 'Shared Memory Throughput')
seen = set()
for r in rows[1:]:
    d = dict(zip(h, r))
    k = d.get('Metric Name')
    if k in want and k not in seen:
        seen.add(k)
        print(f"{k:40s} {d['Metric Value']} {d['Metric Unit']}")
src = gzip.open(pre + ".source.csv.gz", "rt").read()
rows = list(csv.reader(io.StringIO(src)))
i0 = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
hdr = rows[i0]; data = rows[i0 + 1:]
ia = hdr.index("Instructions Executed"); isrc = hdr.index("Source"); ith = hdr.index("Avg. Threads Executed")
ist = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[ia] or 0) for r in data); tst = sum(float(r[ist] or 0) for r in data) or 1
blocks = []; cur = None
for k, r in enumerate(data):
    n = float(r[ia] or 0)
    if cur and cur['n'] == n:
        cur['cnt'] += 1; cur['st'] += float(r[ist] or 0); cur['last'] = r[isrc]; cur['ops'].append(r[isrc].split()[0] if r[isrc].split() else '')
    else:
        cur = {'start': k, 'n': n, 'cnt': 1, 'first': r[isrc], 'last': r[isrc], 'thr': r[ith], 'st': float(r[ist] or 0),
               'ops': [r[isrc].split()[0] if r[isrc].split() else '']}
        blocks.append(cur)
for b in blocks:
    if b['n'] * b['cnt'] / tot > mn or b['st'] / tst > mn:
        print(f"{b['start']:5d} n={int(b['n']):>9d} x{b['cnt']:3d} {b['n']*b['cnt']/tot*100:5.1f}% stall {b['st']/tst*100:5.1f}% "
              f"thr={b['thr']:>5s} | {b['first'].strip()[:45]} .. {b['last'].strip()[:35]}")
print("total instructions", tot)
