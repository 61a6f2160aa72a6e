"""Per-phase stall-reason samples of the segmented kernel (development):
    python tools/ncu_phase_stalls.py report.ncu-rep"""
import csv, collections, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
R = ["stall_wait", "stall_short_sb", "stall_math", "stall_not_selected", "stall_selected", "stall_long_sb",
     "stall_mio", "stall_branch_resolving", "stall_dispatch", "stall_no_inst", "stall_barrier"]
def phase(f, ln):
    if "ffs_warp_kernel" not in f: return "other:" + f.split("/")[-1]
    if 476 <= ln <= 632: return "draw(scan/search)"
    if 634 <= ln <= 714: return "gj"
    if 720 <= ln <= 775: return "init/sample"
    if 776 <= ln <= 869: return "contraction"
    if 870 <= ln <= 1080: return "in-block"
    return "other"
agg = collections.defaultdict(lambda: collections.Counter())
fname = ""; ix = None
for r in rows:
    if r and r[0] == "Line No": ix = {h: i for i, h in enumerate(r)}; continue
    if r and r[0] == "File Path": fname = r[1]; continue
    if ix and r and r[0].isdigit():
        p = phase(fname, int(r[0]))
        for k in R:
            try: agg[p][k] += int(r[ix[k]] or 0)
            except (ValueError, KeyError): pass
tot = sum(sum(c.values()) for c in agg.values())
print("%-22s %6s " % ("phase", "all%") + " ".join("%7s" % k.replace("stall_", "")[:7] for k in R))
for p, c in sorted(agg.items(), key=lambda x: -sum(x[1].values())):
    s = sum(c.values())
    print("%-22s %6.1f " % (p[:22], 100 * s / tot) + " ".join("%7.1f" % (100 * c[k] / tot) for k in R))
