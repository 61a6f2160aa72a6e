"""Small instances of every libffs path, for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): python tools/san_run.py   (each call checked against the oracle where cheap)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import ref  # noqa: E402
from paper_2109_07358_b200 import ffs, inputs  # noqa: E402

dev = torch.device("cuda", 0)
ffs.set_option("graph", float(os.environ.get("SAN_GRAPH", "1")))


def check(U, uni, Np, gpos, what):
    rpos = ref.sample(U, uni, Np=Np)
    bad = int((gpos != rpos).any(axis=1).sum())
    print(f"{what}: {bad} differing samples of {len(rpos)}", flush=True)


for (L, N, Np, M, cplx, what, opts) in [
    (16, 4, 4, 64, False, "seg G=4 (tiny)", {}), (256, 32, 32, 64, False, "seg G=32 (dw)", {}),
    (300, 33, 33, 16, False, "CTA owner", {}), (100, 20, 20, 16, True, "warp owner complex", {}),
    (2100, 40, 40, 4, False, "cluster", {"tile_gram": 0}),
    (2100, 258, 258, 6, False, "block-step dense (Ozaki 8, Gram draws, paired GJ)", {}),
    (2100, 258, 258, 4, True, "block-step dense complex", {}),
    (2100, 258, 258, 4, False, "block-step dense, direct draws, single GJ", {"gram_draw": 0, "gj_pair": 0}),
    (2100, 300, 43, 6, False, "block-step marginal (odd N')", {"tile_gram": 0}),
    (1024, 64, 16, 64, False, "tile-Gram flat, half-warp owners", {}),
    (2100, 300, 43, 16, False, "tile-Gram blocked", {}),
    (2500, 40, 32, 16, True, "tile-Gram complex", {}),
    (40000, 24, 8, 16, False, "tile-Gram, chunked row scan", {}),
    (20000, 16, 8, 16, True, "tile-Gram complex, chunked row scan", {}),
]:
    ffs.reset_options()
    ffs.set_option("graph", float(os.environ.get("SAN_GRAPH", "1")))
    for k, v in opts.items():
        ffs.set_option(k, float(v))
    U = inputs.random_orthonormal(L, N, L + N, complex_=cplx)
    uni = inputs.uniforms(M, Np, 5)
    pos = ffs.ffs_sample_marginal(torch.from_numpy(U).to(dev), torch.from_numpy(uni).to(dev), Np)
    check(U, uni, Np, pos.cpu().numpy(), what)
ffs.reset_options()
ffs.set_option("graph", float(os.environ.get("SAN_GRAPH", "1")))

V, lam = inputs.build_lensemble(L=300, D=40, n_mean=12, seed=3)
uni = inputs.lens_uniforms(16, 40, 8)
pos, cnt, _ = ffs.ffs_sample_lensemble(torch.from_numpy(V).to(dev), torch.from_numpy(lam).to(dev),
                                       torch.from_numpy(uni).to(dev))
rp, rc, _ = ref.sample_lensemble(V, lam, uni)
print("lensemble:", int((pos.cpu().numpy() != rp).any(axis=1).sum()), "differing", flush=True)

U = inputs.random_orthonormal(500, 12, 4)
uni = inputs.metro_uniforms(16, 12, 9, 3)
pos, _ = ffs.ffs_sample_metropolis(torch.from_numpy(U).to(dev), torch.from_numpy(uni).to(dev), 12, 9)
rp, _ = ref.sample_metropolis(U, uni, 12, 9)
print("metropolis:", int((pos.cpu().numpy() != rp).any(axis=1).sum()), "differing", flush=True)

U = inputs.random_orthonormal(64, 8, 6)
uni = inputs.uniforms(64, 8, 7)
pos = ffs.ffs_sample(torch.from_numpy(U).to(dev), torch.from_numpy(uni).to(dev))
occ = ffs.ffs_occupation(pos, 64)
pair = ffs.ffs_pair_occupation(pos, 32)
res, dc = ffs.ffs_gutzwiller_reweight(pos, 64, 0.7)
torch.cuda.synchronize()
print("observables ok:", int(occ.sum().item()) == 64 * 8, flush=True)
