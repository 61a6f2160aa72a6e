#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/ncu_w; mkdir -p $O
python tools/run_once.py dpp 1 > /dev/null 2>&1
FFS_OPTS=gemm_2sm=2 timeout 900 ncu --set full --clock-control none -k regex:ffs_ozaki_gemm2w_kernel -s 60 -c 1 -o $O/full_ozaki2w_dpp \
  python tools/run_once.py dpp 2 > $O/full_ozaki2w_dpp.log 2>&1
ncu -i $O/full_ozaki2w_dpp.ncu-rep --page raw --csv > $O/full_ozaki2w_dpp_raw.csv 2>/dev/null
rm -f $O/*.ncu-rep
python tools/ncu_rawcsv.py $O/full_ozaki2w_dpp_raw.csv
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/ncu_w/full_ozaki2w_dpp_raw.csv")))
h, u, v = rows[0], rows[1], rows[-1]
for k in ("sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_uniform.sum", "l1tex__data_pipe_lsu_wavefronts.sum", "smsp__inst_executed_pipe_tc.sum", "lts__t_sectors_srcunit_tex_op_read.sum", "sm__sass_inst_executed_op_shared_ld.sum"):
    if k in h:
        print(k, v[h.index(k)], u[h.index(k)])
for i, k in enumerate(h):
    if "tensor" in k and "pct" in k:
        print(k, v[i])
PY
