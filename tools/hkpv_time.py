"""FFS vs modified-HKPV on one GPU (development; bench.py extensions has the full table):
python tools/hkpv_time.py dw anderson ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2109_07358_b200 import ffs, inputs  # noqa: E402


def t(fn, k=3):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / k


for name in sys.argv[1:]:
    cfg = inputs.CONFIGS[name]
    U = torch.from_numpy(inputs.build_u(cfg)).cuda()
    uni = inputs.uniforms(cfg.M, cfg.N, 4000)
    ud = torch.from_numpy(uni).cuda()
    us = torch.from_numpy(np.ascontiguousarray(uni[:, cfg.N:])).cuda()
    w1, w2 = ffs.Workspace("cuda"), ffs.Workspace("cuda")
    a = t(lambda: ffs.ffs_sample(U, ud, workspace=w1))
    b = t(lambda: ffs.ffs_sample_hkpv(U, us, workspace=w2))
    print(f"{name}: ffs {a:.2f} ms, hkpv {b:.2f} ms, ratio {b / a:.2f}", flush=True)
