"""Time ffs_sample_marginal on a random orthonormal U (FFS_COMPLEX=1: complex): python tools/shape_time.py L N Np M [opt=val ...] [--- opt=val ...]
Each '---'-separated option group is timed in turn (3 reps after 2 warm-ups, CUDA events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2109_07358_b200 import ffs, inputs

cplx = os.environ.get("FFS_COMPLEX", "0") == "1"
L, N, Np, M = (int(a) for a in sys.argv[1:5])
groups, cur = [], []
for a in sys.argv[5:]:
    if a == "---":
        groups.append(cur); cur = []
    else:
        cur.append(a)
groups.append(cur)
U = torch.from_numpy(inputs.random_orthonormal(L, N, 7 + L + N, complex_=cplx)).cuda()
u = torch.from_numpy(inputs.uniforms(M, Np, 11)).cuda()
ws = ffs.Workspace("cuda")
for g in groups:
    ffs.reset_options()
    for kv in g:
        k, v = kv.split("=")
        ffs.set_option(k, float(v))
    for _ in range(2):
        ffs.ffs_sample_marginal(U, u, Np, workspace=ws)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); ffs.ffs_sample_marginal(U, u, Np, workspace=ws); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"L={L} N={N} Np={Np} M={M}{' complex' if cplx else ''} {' '.join(g) or 'default'}: {min(ts):.3f} ms", flush=True)
