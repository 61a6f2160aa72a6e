"""Executed warp-instructions per sample by SASS opcode from an ncu report (development):
python tools/ncu_opcodes.py report.ncu-rep [M] [addr_lo addr_hi]"""
import csv, subprocess, sys, collections
rep = sys.argv[1]; M = float(sys.argv[2]) if len(sys.argv) > 2 else 65536
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr = rows[1]; ix = {h: i for i, h in enumerate(hdr)}
c = collections.Counter()
for r in rows[2:]:
    if len(r) < len(hdr): continue
    s = r[ix["Source"]].strip()
    if s.startswith("@"): s = s.split(None, 1)[1] if " " in s else s
    op = s.split()[0] if s else "?"
    try: c[op] += int(r[ix["Instructions Executed"]] or 0)
    except ValueError: pass
tot = sum(c.values())
print(f"total {tot / M:.0f} per sample")
for op, v in c.most_common(40):
    print(f"  {op:22s} {v / M:8.0f}  {100 * v / tot:5.1f}%")
