#!/bin/bash
# Round-2 ncu evidence: launch lists (durations; cold, serialised) of the bench headline command
# and of every workload, plus one `--set full` capture of each dominant kernel.
cd $GRAFT_REPO_ROOT
O=gpurun_out/ncu_r2; mkdir -p $O
python tools/run_once.py dpp 1 > /dev/null 2>&1   # builds/caches inputs
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_dpp_bench.csv \
  python bench.py --no-sweep --no-cpu --steps 2 --warmup 3 > $O/launches_dpp_bench.log 2>&1
for w in tiny dw anderson anderson:marginal peierls dpp:marginal lens metro gutzwiller; do
  f=$(echo $w | tr ':' '_')
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$f.csv \
    python tools/run_once.py $w 2 > $O/launches_$f.log 2>&1
done
full() {  # name workload kernel-regex skip
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$3 -s $4 -c 1 -o $O/full_$1 \
    python tools/run_once.py $2 2 > $O/full_$1.log 2>&1
  ncu -i $O/full_$1.ncu-rep --page raw --csv > $O/full_$1_raw.csv 2>/dev/null
  ncu -i $O/full_$1.ncu-rep --page details --csv > $O/full_$1_details.csv 2>/dev/null
  ncu -i $O/full_$1.ncu-rep --page source --csv --print-source sass > $O/full_$1_sass.csv 2>/dev/null
  gzip -f $O/full_$1_sass.csv
  rm -f $O/full_$1.ncu-rep
}
full ozaki8_dpp dpp ffs_ozaki_gemm_kernel 60
full step_dpp dpp "ffs_cluster_kernel" 100
full gj_dpp dpp ffs_dense_gj_kernel 100
full seg_dw dw ffs_seg_kernel 1
full sample_anderson anderson ffs_sample_kernel 1
full stepm_dppm dpp:marginal ffs_cluster_kernel 4
full sample_andersonm anderson:marginal ffs_sample_kernel 1
full lens lens ffs_sample_kernel 1
full metro metro ffs_metro_kernel 1
full gutz gutzwiller ffs_gutzwiller_kernel 1
full ozaki8_peierls peierls ffs_ozaki_gemm_kernel 60
ls -la $O
