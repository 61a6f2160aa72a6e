"""profiles/roofline_r02.json from the round-2 ncu evidence (profiles/r02/final/): per workload the DRAM
traffic of its dominant kernel (dram__bytes_read.sum + dram__bytes_write.sum, one launch, --set full)
and, for the dense path, the Ozaki GEMM's share of the path (launch list) and INT8-pipe activity.
    python tools/make_roofline_json.py [dir]"""
import collections, csv, json, os, sys

D = sys.argv[1] if len(sys.argv) > 1 else "profiles/r02/final"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def raw(name):
    rows = list(csv.reader(open(os.path.join(D, f"full_{name}_raw.csv"))))
    h, v = rows[0], rows[-1]
    d = {}
    for k, x in zip(h, v):
        try:
            d[k] = float(x.replace(",", ""))
        except ValueError:
            d[k] = x
    return d


def to_bytes(d, key):
    # the raw page prints scaled units in row 2; re-read them
    rows = list(csv.reader(open(d["_path"])))
    unit = rows[1][rows[0].index(key)]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[unit]
    return d[key] * scale


def load(name):
    d = raw(name)
    d["_path"] = os.path.join(D, f"full_{name}_raw.csv")
    return d


def shares(name):
    rows = list(csv.reader(open(os.path.join(D, f"launches_{name}.csv"))))
    hdr, agg = None, collections.defaultdict(float)
    for r in rows:
        if r and r[0] == "ID":
            hdr = {h: i for i, h in enumerate(r)}
            continue
        if hdr and len(r) > 5 and r[hdr["Metric Name"]] == "gpu__time_duration.sum":
            agg[r[hdr["Kernel Name"]]] += float(r[hdr["Metric Value"]].replace(",", ""))
    tot = sum(agg.values())
    return {k: v / tot for k, v in agg.items()}


SRC = "ncu --set full --clock-control none, one launch (tools/gpu_r2_final_ncu.sh; profiles/r02/final/full_*_raw.csv): dram__bytes_read.sum + dram__bytes_write.sum of "
out = {}
for wl, cap in [("dw", "seg_dw"), ("anderson", "sample_anderson"), ("anderson:marginal", "km_andersonm"),
                ("dpp:marginal", "km_dppm"), ("dpp", "ozaki2_dpp"), ("peierls", "ozaki2_peierls")]:
    d = load(cap)
    tr = to_bytes(d, "dram__bytes_read.sum") + to_bytes(d, "dram__bytes_write.sum")
    out[wl] = {"traffic": tr, "traffic_source": SRC + str(d.get("Kernel Name", cap))}
    if wl in ("dpp", "peierls"):
        sh = shares("dpp_bench" if wl == "dpp" else "peierls")
        g = sum(v for k, v in sh.items() if "ozaki_gemm" in k)
        out[wl]["traffic_source"] += " (the dominant kernel of the path)"
        out[wl]["gemm"] = {
            "kernel": "ffs_ozaki_gemm2w_kernel (tcgen05.mma.cta_group::2.kind::i8, 256 x 128 pair tiles in two passes, TMEM accumulators, TMA)",
            "share_of_path": round(g, 4),
            "int8_pipe_active": d.get("sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active", 0) / 100,
            "tensor_pipe_active": d.get("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
                                        d.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 0)) / 100,
            "launch_ms_cold": d.get("gpu__time_duration.sum"),
            "path_shares": {k[:60]: round(v, 4) for k, v in sorted(sh.items(), key=lambda kv: -kv[1])[:8]},
            "source": f"{D}/full_{cap}_raw.csv, {D}/launches_{'dpp_bench' if wl == 'dpp' else 'peierls'}.csv",
        }
json.dump(out, open(os.path.join(ROOT, "profiles", "roofline_r02.json"), "w"), indent=1)
print(json.dumps(out, indent=1)[:3000])
