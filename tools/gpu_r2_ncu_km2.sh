#!/bin/bash
# source-level stall profile of the tile-Gram kernel (C3 marginal, C5 marginal)
cd $GRAFT_REPO_ROOT
O=gpurun_out/ncu_km; mkdir -p $O
python tools/run_once.py dpp:marginal 1 > /dev/null 2>&1
for w in anderson:marginal; do
  f=$(echo $w | tr ':' '_')
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffs_kmarg_kernel -s 1 -c 1 -o $O/src_$f \
    python tools/run_once.py $w 2 > $O/src_$f.log 2>&1
  python tools/ncu_top_lines.py $O/src_$f.ncu-rep 45 > $O/src_${f}_toplines.txt 2>&1
  ncu -i $O/src_$f.ncu-rep --page raw --csv > $O/src_${f}_raw.csv 2>/dev/null
  rm -f $O/src_$f.ncu-rep
done
cat $O/src_anderson_marginal_toplines.txt
