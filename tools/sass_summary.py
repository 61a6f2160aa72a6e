"""Summarise an ncu SASS source page (csv): executed instructions and stall samples by opcode."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
ex = collections.Counter(); st = collections.Counter(); tot_ex = 0; tot_st = 0
for r in data:
    if len(r) < len(hdr): continue
    op = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else "?"
    if op.startswith("@"): op = r[ix["Source"]].split()[1]
    op = op.split(".")[0]
    e = int(r[ix["Instructions Executed"]] or 0); s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    ex[op] += e; st[op] += s; tot_ex += e; tot_st += s
print("total executed", tot_ex, "stall samples", tot_st)
for op, e in ex.most_common(25):
    print(f"{op:10s} exec {e:12d} ({100*e/tot_ex:5.1f}%)  stall {100*st[op]/max(tot_st,1):5.1f}%")
if len(sys.argv) > 2:
    # stall reasons columns
    cols = [h for h in hdr if h.startswith("stall_")]
    agg = {c: sum(float(r[ix[c]] or 0) for r in data if len(r) >= len(hdr)) for c in cols}
    for c, v in sorted(agg.items(), key=lambda kv: -kv[1])[:12]:
        print(f"{c:30s} {v:12.0f}")
