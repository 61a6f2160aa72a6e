#!/bin/bash
cd $GRAFT_REPO_ROOT
python tools/run_once.py dpp 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ll_dpp.csv python tools/run_once.py dpp 1 > /dev/null 2>&1
python tools/launch_share.py gpurun_out/ll_dpp.csv > gpurun_out/ll_dpp.txt; head -9 gpurun_out/ll_dpp.txt
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/ll_dpp.csv")))
hdr = None
out = {}
for r in rows:
    if r and r[0] == "ID":
        hdr = {h: i for i, h in enumerate(r)}; continue
    if hdr and len(r) > 5 and ("gj2" in r[hdr["Kernel Name"]] or "dense_gj_kernel" in r[hdr["Kernel Name"]]):
        out.setdefault((r[hdr["ID"]], r[hdr["Kernel Name"]][:40], r[hdr["Grid Size"]]), {})[r[hdr["Metric Name"]]] = (r[hdr["Metric Value"]], r[hdr["Metric Unit"]])
for k in list(out)[-8:]:
    print(k, out[k])
PY
