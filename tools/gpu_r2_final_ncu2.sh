#!/bin/bash
# Re-capture of the kernels changed after gpu_r2_final_ncu.sh (32-byte U^T loads): launch lists of the two
# marginals and C3, one `--set full` capture of each of their dominant kernels.
cd $GRAFT_REPO_ROOT
O=gpurun_out/ncu_final; mkdir -p $O
for w in anderson anderson:marginal dpp:marginal; do
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
full sample_anderson anderson ffs_sample_kernel 1
full km_andersonm anderson:marginal ffs_kmarg_kernel 1
full km_dppm dpp:marginal ffs_kmarg_kernel 1
ls -la $O | tail -12
