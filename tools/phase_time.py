"""development: per-phase clock64 accounting of the segmented warp kernel (FFS_DEBUG_SKIP=8)."""
import ctypes, os, sys
os.environ["FFS_DEBUG_SKIP"] = "8"
import numpy as np, torch
from paper_2109_07358_b200 import ffs, inputs
L = ffs.load()
L.ffs_dev_timing.argtypes = [ctypes.c_void_p, ctypes.c_int]
cfg = inputs.CONFIGS["dw"]
U = inputs.build_u(cfg); uni = inputs.workload_uniforms(cfg)
Ud = torch.from_numpy(U).cuda(); ud = torch.from_numpy(uni).cuda()
ws = ffs.Workspace()
L.ffs_dev_timing(None, 1)
ffs.ffs_sample(Ud, ud, workspace=ws); torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 8)()
L.ffs_dev_timing(None, 1)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); ffs.ffs_sample(Ud, ud, workspace=ws); e1.record(); torch.cuda.synchronize()
L.ffs_dev_timing(buf, 1)
ms = e0.elapsed_time(e1)
tot = sum(buf[:3])
sps = cfg.M * cfg.N
names = ["gemm+init", "steps", "gj", "owner", "extract", "rcp", "col+nextdraw"]
if os.environ.get("FFS_WARP_VARIANT", "").startswith("pc"):
    names = ["prod_wait", "prod_gj", "prod_gemm", "cons_wait", "cons_steps"]
print(f"{os.environ.get('FFS_WARP_VARIANT','default')}: {ms:.3f} ms; cycles per sample-step (sum over warps / sample-steps):",
      {k: round(buf[i] / sps, 1) for i, k in enumerate(names)})
