"""Quick CUDA-event timing of ffs_sample on the registered configs (development aid)."""
import sys, time, json
import numpy as np
import torch
from paper_2109_07358_b200 import ffs, inputs

names = sys.argv[1:] or ["tiny", "dw", "anderson"]
for name in names:
    marg = name.endswith(":m")
    cfg = inputs.CONFIGS[name.split(":")[0]]
    U = inputs.build_u(cfg)
    uni = inputs.workload_uniforms(cfg, marg)
    import os
    if os.environ.get("FFS_QT_M"):
        uni = uni[: int(os.environ["FFS_QT_M"])]
    Np = cfg.marginal_Np if marg else cfg.N
    Ud = torch.from_numpy(U).cuda(); ud = torch.from_numpy(uni).cuda()
    ws = ffs.Workspace()
    f = (lambda: ffs.ffs_sample_marginal(Ud, ud, Np, workspace=ws))
    for _ in range(2): f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    M = uni.shape[0]; L = cfg.L; fac = 4 if np.iscomplexobj(U) else 1
    flops = fac * (L * Np**2 + Np**3) * M
    print(json.dumps({"cfg": name, "ms": ms, "samples_per_s": M / ms * 1e3, "paper_gflops": flops / ms / 1e6,
                      "frac_fp64_36.9": flops / ms / 1e9 / 36.9}), flush=True)
