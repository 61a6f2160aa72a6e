#!/bin/bash
# the driver's bench command (default flags) + the reference arm
cd $GRAFT_REPO_ROOT
timeout 3000 python bench.py > gpurun_out/bench_r02_default.json 2> gpurun_out/bench_r02_default.err
echo "bench rc=$?"
tail -c 600 gpurun_out/bench_r02_default.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_r02_default.json").read().strip().splitlines()[-1])
print("headline", d["config"]["workload"], d["value"], d["ms_per_step"], d["roofline"]["frac"], d["clocks"])
for k, v in d["sweep"].items():
    print(k, f"{v['ms_per_step']:.3f} ms kernel {v['kernel_ms']:.3f} frac {v['frac']:.3f} e2e {v['e2e']['value']:.4g} cpu {v.get('cpu_baseline',{}).get('value')}")
for k, v in d["extensions"].items():
    if k != "hkpv_comparator":
        print(k, v["ms_per_step"], v.get("frac"))
    else:
        for kk, vv in v.items():
            print("hkpv", kk, f"ffs {vv['ffs_ms']:.3f} hkpv {vv['hkpv_ms']:.3f} ratio {vv['time_ratio_hkpv_over_ffs']:.2f}")
PY
