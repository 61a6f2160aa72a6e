"""development: per-phase cycles of the cluster kernel (thread 0 of every CTA; ffs_dev_timing)."""
import ctypes, os, sys
import numpy as np, torch
from paper_2109_07358_b200 import ffs, inputs
name = sys.argv[1] if len(sys.argv) > 1 else "dpp:m"
Mq = int(sys.argv[2]) if len(sys.argv) > 2 else 240
L = ffs.load()
L.ffs_dev_timing.argtypes = [ctypes.c_void_p, ctypes.c_int]
marg = name.endswith(":m"); cfg = inputs.CONFIGS[name.split(":")[0]]
U = torch.from_numpy(inputs.build_u(cfg)).cuda()
uni = torch.from_numpy(inputs.workload_uniforms(cfg, marg)[:Mq]).cuda()
Np = cfg.marginal_Np if marg else cfg.N
ws = ffs.Workspace()
ffs.ffs_sample_marginal(U, uni, Np, workspace=ws); torch.cuda.synchronize()
L.ffs_dev_timing(None, 1)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); ffs.ffs_sample_marginal(U, uni, Np, workspace=ws); e1.record(); torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 8)()
L.ffs_dev_timing(buf, 1)
ms = e0.elapsed_time(e1)
ctas = 120
per = [buf[q] / ctas for q in range(8)]
nd = Mq / 15 * Np
print("per draw: pre-barrier1 %.0f, barrier1 %.0f, select+push %.0f, barrier2 %.0f, update %.0f" % tuple(per[q] / nd for q in range(3, 8)))
print(f"{name} M={Mq}: {ms:.2f} ms; cycles per CTA: contraction {per[0]:.3g}, draws {per[1]:.3g}, GJ {per[2]:.3g};"
      f" per draw {per[1] / (Mq / 15) / Np:.0f}")
