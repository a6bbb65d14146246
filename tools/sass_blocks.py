"""Instruction share per basic block of an ncu capture (development aid):
python tools/sass_blocks.py report.ncu-rep [min_share]"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]; data = rows[2:]
ia = hdr.index("Instructions Executed"); isrc = hdr.index("Source"); ith = hdr.index("Avg. Threads Executed")
ist = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[ia] or 0) for r in data); tst = sum(float(r[ist] or 0) for r in data) or 1
mn = float(sys.argv[2]) if len(sys.argv) > 2 else 0.005
blocks = []; cur = None
for k, r in enumerate(data):
    n = float(r[ia] or 0)
    if cur and cur['n'] == n:
        cur['cnt'] += 1; cur['st'] += float(r[ist] or 0); cur['last'] = r[isrc]
    else:
        cur = {'start': k, 'n': n, 'cnt': 1, 'first': r[isrc], 'last': r[isrc], 'thr': r[ith], 'st': float(r[ist] or 0)}
        blocks.append(cur)
for b in blocks:
    if b['n'] * b['cnt'] / tot > mn:
        print(f"{b['start']:5d} n={int(b['n']):>9d} x{b['cnt']:3d} {b['n']*b['cnt']/tot*100:5.1f}% stall {b['st']/tst*100:5.1f}% "
              f"thr={b['thr']:>4s} | {b['first'].strip()[:45]} .. {b['last'].strip()[:35]}")
print("total instructions", tot)
