"""Per-CUDA-source-line executed instructions and stall samples from an ncu report
(ncu -i X --page source --csv --print-source cuda,sass)."""
import csv, subprocess, sys, collections
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr = None
agg = collections.OrderedDict()
cur = None
for r in rows:
    if r and r[0] == "Line No":
        hdr = r; ix = {h: i for i, h in enumerate(hdr)}; continue
    if hdr is None or len(r) < 8: continue
    if r[0]:
        cur = (int(r[0]), r[1][:100]); agg.setdefault(cur, [0, 0]); continue
    if cur is None: continue
    try:
        agg[cur][0] += int(r[7] or 0); agg[cur][1] += int(r[4] or 0)
    except ValueError:
        pass
tot = sum(v[0] for v in agg.values()) or 1; tots = sum(v[1] for v in agg.values()) or 1
print("total instr", tot, "stall samples", tots)
for (ln, src), (e, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{ln:>4} {100*e/tot:5.1f}% stall {100*s/tots:5.1f}%  {src}")
