"""Block-step schedule scan (development): python tools/theta_scan.py <config> theta1 theta2 ...
Times ffs_sample (CUDA events, 3 reps after 2 warm-up) for each gathered/GEMM crossover theta."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2109_07358_b200 import ffs, inputs  # noqa: E402

name, _, marg = sys.argv[1].partition(":")
cfg = inputs.CONFIGS[name]
U = torch.from_numpy(inputs.build_u(cfg)).cuda()
u = torch.from_numpy(inputs.workload_uniforms(cfg, bool(marg))).cuda()
Np = cfg.marginal_Np if marg else cfg.N
ws = ffs.Workspace("cuda")
for th in sys.argv[2:]:
    key, _, val = th.partition("=")
    if val:
        ffs.set_option(key, float(val))
    elif key != "-":
        ffs.set_option("dense_theta", float(key))
    for _ in range(2):
        ffs.ffs_sample_marginal(U, u, Np, workspace=ws)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ffs.ffs_sample_marginal(U, u, Np, workspace=ws)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(name, th, f"{min(ts):.3f} ms", flush=True)
