"""development: per-phase cycles of the dense path's step kernel (thread 0 of every CTA; ffs_dev_timing)."""
import ctypes, sys
import torch
from paper_2109_07358_b200 import ffs, inputs
name = sys.argv[1] if len(sys.argv) > 1 else "dpp"
Mq = int(sys.argv[2]) if len(sys.argv) > 2 else 256
L = ffs.load()
L.ffs_dev_timing.argtypes = [ctypes.c_void_p, ctypes.c_int]
cfg = inputs.CONFIGS[name]
U = torch.from_numpy(inputs.build_u(cfg)).cuda()
uni = torch.from_numpy(inputs.workload_uniforms(cfg, False)[:Mq]).cuda()
Np = cfg.N
ws = ffs.Workspace()
ffs.ffs_sample_marginal(U, uni, Np, workspace=ws); torch.cuda.synchronize()
L.ffs_dev_timing(None, 1)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); ffs.ffs_sample_marginal(U, uni, Np, workspace=ws); e1.record(); torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 8)()
L.ffs_dev_timing(buf, 1)
cs = 8 if cfg.L > 8192 else 4
ctas = Mq * cs * (Np // 8)  # CTA-steps
nd = Mq * cs * Np             # CTA-draws
print(f"{name} M={Mq}: {e0.elapsed_time(e1):.1f} ms (with timing); per CTA-step cycles: panel load {buf[0]/ctas:.0f}, "
      f"draws {buf[1]/ctas:.0f}, rest {buf[2]/ctas:.0f}")
print("per draw: pre-barrier1 %.0f, barrier1 %.0f, select+push %.0f, barrier2 %.0f, update %.0f" % tuple(buf[q] / nd for q in range(3, 8)))
