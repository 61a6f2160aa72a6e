#!/bin/bash
# ncu --set full captures of the tile-Gram marginal kernel (C3 marginal, C5 marginal) and the Gram kernels (C5)
cd $GRAFT_REPO_ROOT
O=gpurun_out/ncu_km; mkdir -p $O
python tools/run_once.py dpp:marginal 1 > /dev/null 2>&1
full() {  # name workload kernel-regex skip
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$3 -s $4 -c 1 -o $O/full_$1 \
    python tools/run_once.py $2 2 > $O/full_$1.log 2>&1
  ncu -i $O/full_$1.ncu-rep --page raw --csv > $O/full_$1_raw.csv 2>/dev/null
  ncu -i $O/full_$1.ncu-rep --page source --csv --print-source sass > $O/full_$1_sass.csv 2>/dev/null
  gzip -f $O/full_$1_sass.csv
  rm -f $O/full_$1.ncu-rep
}
full km_andersonm anderson:marginal ffs_kmarg_kernel 1
full km_dppm dpp:marginal ffs_kmarg_kernel 1
full gram_dpp dpp "ffs_gram_kernel" 60
full gramdraw_dpp dpp "ffs_gram_draw_kernel" 60
ls -la $O
