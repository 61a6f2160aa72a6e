import numpy as np, torch, os
from oracle import ref
from paper_2109_07358_b200 import ffs, inputs
L,N=2048,256
U = inputs.random_orthonormal(L, N, 1000 + L + N, complex_=True)
uni = inputs.uniforms(60, N, L * 7 + N)
Ud=torch.from_numpy(U).cuda(); ud=torch.from_numpy(uni).cuda()
pos, flags, w = ffs.ffs_debug_trace(Ud, ud, N, 2)
torch.cuda.synchronize()
gw=w.cpu().numpy(); gp=pos.cpu().numpy()
rp, rw = ref.weights(U, uni[:2], Np=N)
print("pos eq first steps", (gp[0][:20]==rp[0][:20]).astype(int))
for k in range(0,24):
    e=np.abs(gw[0,k]-rw[0,k]).max()/rw[0,k].max()
    print(k, e)
