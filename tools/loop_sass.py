"""Print the hot loops (backward branches enclosing MUFU.EX2) of one kernel of a cubin with their
instruction counts (development aid).  usage: python tools/loop_sass.py CUBIN FUNC_SUBSTRING [-v]"""
import re, subprocess, sys
out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if sys.argv[2] not in name:
        continue
    ins = []
    for line in f.split("\n"):
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    addr = {a: i for i, (a, _) in enumerate(ins)}
    print(name[-60:], len(ins), "instructions")
    for i, (a, t) in enumerate(ins):
        m = re.search(r"BRA (0x[0-9a-f]+)", t)
        if m and int(m.group(1), 16) < a:
            j = addr.get(int(m.group(1), 16))
            if j is None: continue
            body = [x for _, x in ins[j:i + 1]]
            if any("MUFU" in x or "FFMA2" in x for x in body) and len(body) < 400:
                ops = {}
                for x in body:
                    op = x.split()[0] if not x.startswith("@") else x.split()[1]
                    ops[op.split(".")[0]] = ops.get(op.split(".")[0], 0) + 1
                print(f"  loop {ins[j][0]:#x}-{a:#x}: {len(body)} instr  " + " ".join(f"{k}:{v}" for k, v in sorted(ops.items(), key=lambda kv: -kv[1])))
                if "-v" in sys.argv:
                    for x in body: print("     ", x)
