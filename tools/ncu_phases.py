"""Per-phase executed warp-instructions, smem wavefronts (and bank-conflict excess) and stall
samples of the segmented kernel from an ncu report with source (development):
    python tools/ncu_phases.py report.ncu-rep [M]"""
import csv, subprocess, sys, collections, re
rep = sys.argv[1]
M = float(sys.argv[2]) if len(sys.argv) > 2 else 65536
src = open("paper_2109_07358_b200/csrc/ffs_warp_kernel.cuh").read().splitlines()
def find(pat, start=0):
    for i in range(start, len(src)):
        if re.search(pat, src[i]): return i + 1
    raise KeyError(pat)
body = find(r"void ffs_seg_body")
ranges = [
    ("draw", find(r"^__device__ __forceinline__ double fast_rcp"), find(r"^// Rare paths for one segment")),
    ("gj", find(r"seg_gj_flat\(const double"), body),
    ("init/sample", body, find(r"a3 panel", body)),
    ("gemm+panel", find(r"a3 panel", body), find(r"a4/a5", body)),
    ("steps", find(r"a4/a5", body), find(r"Gauss-Jordan update of W with", body)),
    ("gj", find(r"Gauss-Jordan update of W with", body), find(r"a6: positions", body)),
    ("output", find(r"a6: positions", body), len(src) + 1),
]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
ix = None; fname = ""
keys = ["Instructions Executed", "L1 Wavefronts Shared", "L1 Wavefronts Shared Excessive", "Warp Stall Sampling (All Samples)"]
agg = collections.defaultdict(lambda: [0, 0, 0, 0])
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1]; continue
    if r and r[0] == "Line No":
        ix = {h: i for i, h in enumerate(r)}  # first occurrence of each name
        ix = {}
        for i, h in enumerate(r):
            ix.setdefault(h, i)
        continue
    if ix is None or not r or not r[0]: continue
    try: ln = int(r[0])
    except ValueError: continue
    ph = "other:" + fname.split("/")[-1]
    if fname.endswith("ffs_warp_kernel.cuh"):
        ph = "other"
        for name, a, b in ranges:
            if a <= ln < b: ph = name; break
    for j, k in enumerate(keys):
        try: agg[ph][j] += int(r[ix[k]] or 0)
        except (ValueError, KeyError): pass
tot = [sum(v[j] for v in agg.values()) or 1 for j in range(4)]
print(f"per sample: {tot[0] / M:.0f} warp-instr, {tot[1] / M:.0f} smem wavefronts ({tot[2] / M:.0f} conflict excess)")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"  {k:28s} instr {v[0] / M:7.0f} ({100 * v[0] / tot[0]:4.1f}%)  smem {v[1] / M:6.0f} (+{v[2] / M:5.0f} conflicts)  stall {100 * v[3] / tot[3]:4.1f}%")
