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


# pair correlations of the GPU samples against the projection-DPP closed form
# <n_x n_y> = K_xx K_yy - |K_xy|^2 (K = U U^dagger); for the marginal of N' < N particles the first N'
# picks of an exchangeable order give the factor N'(N'-1) / (N(N-1)). Counted on the device
# (ffs_pair_occupation) over the window of the W sites with the largest occupation; z-test with a
# Bonferroni bound where the expected count is >= 50, pooled Poisson check for the rest.
@pytest.mark.parametrize("name,marginal", [("dw", False), ("anderson", True), ("dpp", True)])
def test_pair_correlations_full_size(name, marginal):
    from scipy import stats
    ffs = _ffs()
    cfg = inputs.CONFIGS[name]
    U = inputs.build_u(cfg)
    Np = cfg.marginal_Np if marginal else cfg.N
    M = cfg.marginal_M if marginal else cfg.M
    uni = inputs.uniforms(M, Np, cfg.uniform_seed + 700)
    pos = ffs.ffs_sample_marginal(torch.from_numpy(U).cuda(), torch.from_numpy(uni).cuda(), Np)
    torch.cuda.synchronize()
    Kd = np.sum(np.abs(U) ** 2, axis=1)
    W = 64
    sites = np.sort(np.argsort(-Kd)[:W])            # the W most occupied sites, relabelled 0..W-1
    hp = pos.cpu().numpy()
    relabel = np.full(cfg.L, -1, dtype=np.int32)
    relabel[sites] = np.arange(W, dtype=np.int32)
    sub = relabel[hp]                               # other sites become -1 (skipped by the observables)
    pair = ffs.ffs_pair_occupation(torch.from_numpy(np.ascontiguousarray(sub)).cuda(), W).cpu().numpy().astype(np.float64)
    Us = U[sites]
    K = Us @ Us.conj().T
    fac = Np * (Np - 1) / (cfg.N * (cfg.N - 1))
    P = fac * (np.outer(np.diag(K).real, np.diag(K).real) - np.abs(K) ** 2)
    iu = np.triu_indices(W, 1)
    p, obs = np.clip(P[iu], 0.0, 1.0), pair[iu]
    big = M * p * (1 - p) >= 50
    if name != "dpp":  # (C5's marginal has no pair with an expected count >= 50 at M = 8192: pooled check only)
        assert big.sum() >= 20, big.sum()
    if big.any():
        z = np.abs(obs[big] / M - p[big]) / np.sqrt(p[big] * (1 - p[big]) / M)
        assert z.max() < stats.norm.isf(1e-3 / (2 * big.sum())), (z.max(), int(big.sum()))
    lam, tot = M * p[~big].sum(), obs[~big].sum()
    if lam > 0:
        assert stats.poisson.sf(tot - 1, lam) > 1e-4 and stats.poisson.cdf(tot, lam) > 1e-4, (tot, lam)


# Large L on the tile-Gram path (L = 65536: 64 rows per lane of the crossing tile, scanned in four
# chunks of 16): single-site occupations of the marginal against the closed form
# <n_x> = (N'/N) K_xx (exchangeable column order). U has a localised envelope, so that a
# few thousand rows around the maxima carry expected counts >= 50. n_x is 0 or 1 per sample and the
# samples are independent, so the count of a site is exactly binomial(M, <n_x>).
@pytest.mark.parametrize("complex_", [False, True])
def test_large_L_marginal_occupations(complex_):
    from scipy import stats
    ffs = _ffs()
    L, N, Np, M = 65536, 32, 8, 65536
    rng = np.random.default_rng(4242 + int(complex_))
    x = np.arange(L)
    env = np.exp(-0.5 * ((x - 30011.0) / 700.0) ** 2) + 0.4 * np.exp(-0.5 * ((x - 51007.0) / 300.0) ** 2) + 1e-3
    A = rng.standard_normal((L, N))
    if complex_:
        A = A + 1j * rng.standard_normal((L, N))
    U, _ = np.linalg.qr(A * env[:, None])
    U = np.ascontiguousarray(U)
    uni = inputs.uniforms(M, Np, 90210 + int(complex_))
    pos, flags = ffs.ffs_sample_marginal(torch.from_numpy(U).cuda(), torch.from_numpy(uni).cuda(), Np, with_flags=True)
    torch.cuda.synchronize()
    assert (flags.cpu().numpy() == 0).all()
    hp = pos.cpu().numpy()
    assert all(len(set(q)) == Np for q in hp[:: M // 512].tolist())
    obs = np.bincount(hp.ravel(), minlength=L).astype(np.float64)
    p = (Np / N) * np.sum(np.abs(U) ** 2, axis=1)
    big = M * p >= 50
    assert big.sum() >= 1000, big.sum()
    z = np.abs(obs[big] - M * p[big]) / np.sqrt(M * p[big] * (1 - p[big]))
    assert z.max() < stats.norm.isf(1e-3 / (2 * big.sum())), (z.max(), int(big.sum()))
    lam, tot = M * p[~big].sum(), obs[~big].sum()
    assert stats.poisson.sf(tot - 1, lam) > 1e-4 and stats.poisson.cdf(tot, lam) > 1e-4, (tot, lam)
    # the z-scores as a whole: mean square 1 up to sampling noise
    assert np.mean(z ** 2) < 1.15, np.mean(z ** 2)
