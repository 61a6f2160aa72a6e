#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python tools/theta_scan.py anderson:marginal - tile_gram=2 > gpurun_out/exp1_anderson_m.log 2>&1
cat gpurun_out/exp1_anderson_m.log
python - <<'PY' > gpurun_out/exp1_kappa.log 2>&1
import torch
from paper_2109_07358_b200 import ffs, inputs
for name in ("dpp", "peierls"):
    cfg = inputs.CONFIGS[name]
    U = torch.from_numpy(inputs.build_u(cfg)).cuda()
    u = torch.from_numpy(inputs.workload_uniforms(cfg, False)).cuda()
    ws = ffs.Workspace("cuda")
    for kap in (1e3, 1e4, 1e5, 1e30):
        ffs.set_option("gram_kappa", kap)
        ffs.ffs_sample(U, u, workspace=ws)
        ffs.ffs_gram_counters(reset=True)
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); ffs.ffs_sample(U, u, workspace=ws); e1.record(); e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        d, f = ffs.ffs_gram_counters()
        print(name, "kappa", kap, f"{min(ts):.1f} ms", "draws", d // 3, "direct", f // 3, flush=True)
PY
cat gpurun_out/exp1_kappa.log
