#!/bin/bash
# round 2: Gram draws -- parity tests, theta scan with the new draws, C3 on the block-step path
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -s -k "dense_path or gram or graph_replay or small_batches" > gpurun_out/gram_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gram_pytest.log
tail -5 gpurun_out/gram_pytest.log
timeout 900 python tools/theta_scan.py dpp 0.15 0.1 0.05 0.02 0 > gpurun_out/gram_theta_dpp.log 2>&1
cat gpurun_out/gram_theta_dpp.log
timeout 900 python tools/theta_scan.py peierls 0.3 0.2 0.1 0.05 0 > gpurun_out/gram_theta_peierls.log 2>&1
cat gpurun_out/gram_theta_peierls.log
timeout 600 python tools/theta_scan.py anderson - dense_min_n=128 dense_min_l=1024 > gpurun_out/gram_anderson.log 2>&1
cat gpurun_out/gram_anderson.log
python - <<'PY' > gpurun_out/gram_counters.log 2>&1
import torch
from paper_2109_07358_b200 import ffs, inputs
for name in ("dpp", "peierls"):
    cfg = inputs.CONFIGS[name]
    U = torch.from_numpy(inputs.build_u(cfg)).cuda()
    u = torch.from_numpy(inputs.workload_uniforms(cfg, False)).cuda()
    ffs.ffs_gram_counters(reset=True)
    ffs.ffs_sample(U, u)
    torch.cuda.synchronize()
    print(name, "gram draws, direct recomputations:", ffs.ffs_gram_counters())
PY
cat gpurun_out/gram_counters.log
