#!/bin/bash
# final round-2 evidence: full GPU suite (normal build + checked build test), default bench, reference arm
cd $GRAFT_REPO_ROOT
timeout 3000 python -m pytest tests -m gpu -x -q -s > gpurun_out/final_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/final_pytest.log
tail -3 gpurun_out/final_pytest.log
timeout 3000 python bench.py > gpurun_out/bench_r02_final.json 2> gpurun_out/bench_r02_final.err
echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_r02_final.json").read().strip().splitlines()[-1])
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
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_r02_reference.json 2>&1
tail -c 400 gpurun_out/bench_r02_reference.json
