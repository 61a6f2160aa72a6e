#!/bin/bash
# Round-2 final ncu evidence: launch lists (durations; cold, serialised) of the bench headline
# command and of every sweep workload, plus one `--set full` capture of each dominant kernel.
cd $GRAFT_REPO_ROOT
O=gpurun_out/ncu_final; mkdir -p $O
python tools/run_once.py dpp 1 > /dev/null 2>&1   # builds/caches inputs
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_dpp_bench.csv \
  python bench.py --no-sweep --no-cpu --steps 2 --warmup 3 > $O/launches_dpp_bench.log 2>&1
for w in tiny dw anderson anderson:marginal peierls dpp:marginal; do
  f=$(echo $w | tr ':' '_')
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$f.csv \
    python tools/run_once.py $w 2 > $O/launches_$f.log 2>&1
done
full() {  # name workload kernel-regex skip
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$3 -s $4 -c 1 -o $O/full_$1 \
    python tools/run_once.py $2 2 > $O/full_$1.log 2>&1
  ncu -i $O/full_$1.ncu-rep --page raw --csv > $O/full_$1_raw.csv 2>/dev/null
  rm -f $O/full_$1.ncu-rep
}
full ozaki2_dpp dpp ffs_ozaki_gemm2w_kernel 60
full gram_dpp dpp "ffs_gram_kernel" 60
full gramdraw_dpp dpp ffs_gram_draw_kernel 60
full gj_dpp dpp ffs_dense_gj_kernel 100
full gj2_dpp dpp ffs_dense_gj2_kernel 50
full step_dpp dpp ffs_cluster_kernel 8
full ozaki2_peierls peierls ffs_ozaki_gemm2w_kernel 30
full gram_peierls peierls "ffs_gram_kernel" 30
full gramdraw_peierls peierls ffs_gram_draw_kernel 30
full seg_dw dw ffs_seg_kernel 1
full sample_anderson anderson ffs_sample_kernel 1
full km_andersonm anderson:marginal ffs_kmarg_kernel 1
full km_dppm dpp:marginal ffs_kmarg_kernel 1
full tilegram_dppm dpp:marginal ffs_tile_gram_u_kernel 1
ls -la $O
