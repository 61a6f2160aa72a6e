"""Device observables (ffs_occupation, ffs_pair_occupation, ffs_gutzwiller_reweight; Supp S5)
against the oracle's plain loops on the same positions: integer counts bit-exact, reweighted
averages within the oracle's recursive-summation bound (the device sums by D-histograms, the oracle
sample by sample)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import ref  # noqa: E402
from paper_2109_07358_b200 import inputs  # noqa: E402

pytestmark = pytest.mark.gpu


def _ffs():
    from paper_2109_07358_b200 import ffs
    return ffs


def _gpu_positions(name, M=None):
    ffs = _ffs()
    cfg = inputs.CONFIGS[name]
    U = inputs.build_u(cfg)
    M = cfg.M if M is None else M
    uni = inputs.uniforms(M, cfg.N, cfg.uniform_seed + 500)
    pos = ffs.ffs_sample(torch.from_numpy(U).cuda(), torch.from_numpy(uni).cuda())
    torch.cuda.synchronize()
    return cfg, U, pos


@pytest.mark.parametrize("name", ["dw", "anderson", "tiny"])
def test_occupation_and_pairs_bitexact(name):
    ffs = _ffs()
    cfg, U, pos = _gpu_positions(name, M=None if name != "anderson" else 4096)
    hp = pos.cpu().numpy()
    occ = ffs.ffs_occupation(pos, cfg.L).cpu().numpy().astype(np.uint64)
    assert (occ == ref.occupation(hp, cfg.L)).all()
    W = min(cfg.L, 96)
    pair = ffs.ffs_pair_occupation(pos, W).cpu().numpy().astype(np.uint64)
    assert (pair == ref.pair_occupation(hp, W)).all()


def test_occupation_of_padded_lensemble_rows():
    ffs = _ffs()
    V, lam = inputs.build_lensemble(L=300, D=40, n_mean=12, seed=3)
    uni = inputs.lens_uniforms(2000, 40, 8)
    pos, cnt, _ = ffs.ffs_sample_lensemble(torch.from_numpy(V).cuda(), torch.from_numpy(lam).cuda(),
                                           torch.from_numpy(uni).cuda())
    occ = ffs.ffs_occupation(pos, 300).cpu().numpy().astype(np.uint64)
    assert (occ == ref.occupation(pos.cpu().numpy(), 300)).all()
    assert int(occ.sum()) == int(cnt.sum().item())


@pytest.mark.parametrize("name,V", [("dw", 0.0), ("dw", 0.8), ("anderson", 2.0), ("tiny", 1.3)])
def test_gutzwiller_matches_oracle(name, V):
    ffs = _ffs()
    cfg, U, pos = _gpu_positions(name, M=None if name != "anderson" else 8192)
    hp = pos.cpu().numpy()
    res, dcount = ffs.ffs_gutzwiller_reweight(pos, cfg.L, V)
    res = res.cpu().numpy()
    want = ref.gutzwiller(hp, cfg.L, V)
    # the oracle sums Ms terms in sample order: recursive-summation error <= (Ms - 1) u relative
    # per sum (u = 2^-53); the quotient of two such sums doubles it; the device sums are exact
    # integer histograms combined over <= N'+1 values of D
    Ms = hp.shape[0] // 2
    np.testing.assert_allclose(res, want, rtol=2 * Ms * 2.0 ** -53 + 1e-14, atol=0)
    # D histogram: the number of doubly occupied sites of every spinful sample, counted directly
    up, dn = hp[0::2], hp[1::2]
    D = np.array([len(set(a) & set(b)) for a, b in zip(up.tolist(), dn.tolist())])
    assert (dcount.cpu().numpy() == np.bincount(D, minlength=cfg.N + 1)).all()
    if V == 0.0:
        assert res[0] == 1.0
