#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/ncu_r2b; mkdir -p $O
python tools/run_once.py dpp 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffs_ozaki_gemm2_kernel -s 60 -c 1 -o $O/full_ozaki2_dpp python tools/run_once.py dpp 2 > $O/full_ozaki2_dpp.log 2>&1
ncu -i $O/full_ozaki2_dpp.ncu-rep --page raw --csv > $O/full_ozaki2_dpp_raw.csv 2>/dev/null
ncu -i $O/full_ozaki2_dpp.ncu-rep --page source --csv --print-source sass > $O/full_ozaki2_dpp_sass.csv 2>/dev/null; gzip -f $O/full_ozaki2_dpp_sass.csv
rm -f $O/full_ozaki2_dpp.ncu-rep
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_dpp.csv python tools/run_once.py dpp 2 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_peierls.csv python tools/run_once.py peierls 2 > /dev/null 2>&1
