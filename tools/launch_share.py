"""Per-kernel launch counts, total/average device time and share from an ncu launch-list CSV
(--metrics gpu__time_duration.sum --csv): python tools/launch_share.py launches.csv"""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if r and r[0] == "ID":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr and r and len(r) > 5 and r[hdr["Metric Name"]] == "gpu__time_duration.sum":
        k = r[hdr["Kernel Name"]][:80]
        agg[k][0] += 1
        agg[k][1] += float(r[hdr["Metric Value"]].replace(",", ""))
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"| {k} | {v[0]} | {v[1] / 1e6:.1f} ms | {100 * v[1] / tot:.1f} % | {v[1] / v[0] / 1e3:.1f} us |")
