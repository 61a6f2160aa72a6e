"""Hot SASS regions from `ncu --page source --csv --print-source sass` dumps (gz ok):
python tools/sass_hot.py x_sass.csv.gz [window]  -- prints executed-instruction and stall shares in windows of N instrs"""
import csv, gzip, sys
path = sys.argv[1]; win = int(sys.argv[2]) if len(sys.argv) > 2 else 24
f = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
rows = list(csv.reader(f))
h = rows[1]; iS = h.index("Warp Stall Sampling (All Samples)"); iI = h.index("Instructions Executed")
ins = [(r[1].strip(), int(r[iS] or 0), int(r[iI] or 0)) for r in rows[2:] if len(r) > iI and r[0].startswith("0x")]
ts = sum(x[1] for x in ins); ti = sum(x[2] for x in ins)
print(f"{len(ins)} SASS instrs, {ti} executed, {ts} stall samples")
for a in range(0, len(ins), win):
    blk = ins[a:a + win]
    s = sum(x[1] for x in blk); i = sum(x[2] for x in blk)
    if s / max(ts, 1) > 0.02 or i / max(ti, 1) > 0.02:
        ops = {}
        for x in blk:
            op = x[0].split()[0] if not x[0].startswith("@") else x[0].split()[1]
            ops[op.split(".")[0]] = ops.get(op.split(".")[0], 0) + 1
        top = sorted(blk, key=lambda x: -x[1])[:2]
        print(f"[{a:5d}] stall {100*s/ts:5.1f}% instr {100*i/ti:5.1f}%  " + " ".join(f"{k}:{v}" for k, v in sorted(ops.items(), key=lambda kv: -kv[1])[:7]) + "  | " + " ; ".join(t[0][:50] for t in top))
