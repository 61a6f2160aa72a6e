"""Top source lines by stall samples (and their instruction share) from an ncu report
(development): python tools/ncu_top_lines.py report.ncu-rep [n]"""
import csv, subprocess, sys
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out)); ix = None; fname = ""; res = []; ts = ti = 0
for r in rows:
    if r and r[0] == "File Path": fname = r[1]; continue
    if r and r[0] == "Line No":
        ix = {}
        for i, h in enumerate(r): ix.setdefault(h, i)
        continue
    if ix is None or not r or not r[0]: continue
    try:
        ln = int(r[0]); st = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0); ins = int(r[ix["Instructions Executed"]] or 0)
    except (ValueError, KeyError):
        continue
    ts += st; ti += ins; res.append((st, ins, fname.split("/")[-1], ln, r[1][:80]))
for st, ins, f, ln, s in sorted(res, reverse=True)[:n]:
    print(f"stall {100 * st / max(ts, 1):5.1f}% instr {100 * ins / max(ti, 1):5.1f}%  {f}:{ln} {s}")
