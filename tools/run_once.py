"""One call of a workload (for ncu captures): python tools/run_once.py <workload> [reps]
workloads: tiny dw anderson anderson:marginal peierls dpp dpp:marginal lens metro gutzwiller"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2109_07358_b200 import ffs, inputs  # noqa: E402

for kv in filter(None, os.environ.get("FFS_OPTS", "").split(",")):  # e.g. FFS_OPTS=gemm_2sm=2,dense_theta=0
    k, v = kv.split("=")
    ffs.set_option(k, float(v))
name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = torch.device("cuda", 0)
if name == "lens":
    V, lam = inputs.build_lensemble()
    uni = inputs.lens_uniforms(inputs.LENS.M, inputs.LENS.D, inputs.LENS.uniform_seed)
    a = [torch.from_numpy(x).to(dev) for x in (V, lam, uni)]
    ws = ffs.Workspace(dev)
    for _ in range(reps):
        ffs.ffs_sample_lensemble(*a, workspace=ws)
elif name == "metro":
    mc = inputs.METRO
    U = torch.from_numpy(inputs.build_box_orbitals(mc.L, mc.N)).to(dev)
    u = torch.from_numpy(inputs.metro_uniforms(mc.M, mc.N, mc.Mc, mc.uniform_seed)).to(dev)
    ws = ffs.Workspace(dev)
    for _ in range(reps):
        ffs.ffs_sample_metropolis(U, u, mc.N, mc.Mc, workspace=ws)
elif name == "gutzwiller":
    cfg = inputs.CONFIGS["dw"]
    pos = ffs.ffs_sample(torch.from_numpy(inputs.build_u(cfg)).to(dev),
                         torch.from_numpy(inputs.workload_uniforms(cfg)).to(dev))
    for _ in range(reps):
        ffs.ffs_gutzwiller_reweight(pos, cfg.L, 1.0)
else:
    base, _, marg = name.partition(":")
    cfg = inputs.CONFIGS[base]
    U = torch.from_numpy(inputs.build_u(cfg)).to(dev)
    u = torch.from_numpy(inputs.workload_uniforms(cfg, bool(marg))).to(dev)
    Np = cfg.marginal_Np if marg else cfg.N
    ws = ffs.Workspace(dev)
    for _ in range(reps):
        ffs.ffs_sample_marginal(U, u, Np, workspace=ws)
torch.cuda.synchronize()
print("done", name)
