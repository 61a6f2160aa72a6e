#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/ll; mkdir -p $O
python tools/run_once.py dpp:marginal 1 > /dev/null 2>&1
for w in anderson:marginal dpp:marginal; do
  f=$(echo $w | tr ':' '_')
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_$f.csv \
    python tools/run_once.py $w 2 > $O/launches_$f.log 2>&1
  python tools/launch_share.py $O/launches_$f.csv 2>&1 | head -12
  grep -v "^==" $O/launches_$f.csv | tail -24 | cut -d, -f5,13,15 | head -30
done
