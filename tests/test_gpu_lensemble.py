"""L-ensemble front end on the GPU (ffs_sample_lensemble) against the oracle
(ref.sample_lensemble) on identical seeded inputs: bit-exact positions and counts (modulo reported
CDF-boundary ties), over every owner variant of the ragged-mode kernel (warp owners with shared or
global V^T, CTA owners of each register class, real and complex), the empty and all-kept spectra,
the L-ensemble law on a tiny kernel, and the full-size `lens` workload on spread samples."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import exact, ref  # noqa: E402
from paper_2109_07358_b200 import inputs  # noqa: E402
from tests.parity import compare_positions  # noqa: E402

pytestmark = pytest.mark.gpu


def _ffs():
    from paper_2109_07358_b200 import ffs
    return ffs


def run_gpu(V, lam, uni):
    ffs = _ffs()
    pos, cnt, flags = ffs.ffs_sample_lensemble(torch.from_numpy(np.ascontiguousarray(V)).cuda(),
                                               torch.from_numpy(lam).cuda(), torch.from_numpy(uni).cuda())
    torch.cuda.synchronize()
    return pos.cpu().numpy(), cnt.cpu().numpy(), flags.cpu().numpy()


def compare(V, lam, uni, gpos, gcnt, rpos, rcnt):
    """Counts bit-exact (the keep rule is an fp64 comparison on both sides); positions bit-exact
    except CDF-boundary ties, checked per sample on its own U_i = V[:, kept] (tests/parity.py)."""
    assert (gcnt == rcnt).all(), np.nonzero(gcnt != rcnt)[0][:5]
    K = V.shape[1]
    ties, exact_rows = 0, 0
    for i in np.nonzero((gpos != rpos).any(axis=1))[0]:
        kept = np.nonzero(uni[i, :K] < lam / (lam + 1.0))[0]
        n = len(kept)
        Ui = V[:, kept]
        row = np.concatenate([uni[i, K:K + n], uni[i, 2 * K:2 * K + n]])[None, :]
        r = compare_positions(Ui, row, gpos[i:i + 1, :n], rpos[i:i + 1, :n], n)
        assert not r["failures"], (i, r["failures"])
        ties += r["ties"]
    exact_rows = len(gpos) - ties
    assert (gpos[np.arange(K)[None, :] >= gcnt[:, None]] == -1).all()
    return exact_rows, ties


SHAPES = [  # (L, K, complex): warp owners (L <= 256 real / 128 complex), CTA owners, ragged tails
    (16, 6, False), (40, 12, False), (100, 30, False), (256, 48, False), (300, 70, False),
    (1024, 256, False), (1500, 40, False), (5000, 24, False),
    (30, 9, True), (128, 40, True), (500, 60, True), (3000, 20, True),
]


@pytest.mark.parametrize("L,K,cplx", SHAPES)
def test_lensemble_shapes_match_oracle(L, K, cplx):
    V, lam = inputs.build_lensemble(L=L, D=K, n_mean=K / 3, seed=L + K, complex_=cplx)
    M = 400 if L * K < 100000 else 120
    uni = inputs.lens_uniforms(M, K, 7 * L + K)
    gpos, gcnt, gfl = run_gpu(V, lam, uni)
    rpos, rcnt, rfl = ref.sample_lensemble(V, lam, uni)
    compare(V, lam, uni, gpos, gcnt, rpos, rcnt)
    assert (gfl == 0).all()
    for p, c in zip(gpos.tolist(), gcnt.tolist()):  # Pauli exclusion within each sample
        assert len(set(p[:c])) == c


def test_lensemble_degenerate_spectra():
    L, K = 300, 20
    V = inputs.random_orthonormal(L, K, 3)
    uni = inputs.lens_uniforms(64, K, 5)
    gpos, gcnt, _ = run_gpu(V, np.zeros(K), uni)
    assert (gcnt == 0).all() and (gpos == -1).all()
    gpos, gcnt, _ = run_gpu(V, np.full(K, 1e300), uni)
    assert (gcnt == K).all()
    # every eigenvector kept: the sample is ffs_sample of V on the same permutation/selection draws
    ffs = _ffs()
    full = ffs.ffs_sample(torch.from_numpy(V).cuda(), torch.from_numpy(np.ascontiguousarray(uni[:, K:])).cuda())
    assert (gpos == full.cpu().numpy()).all()


def test_lensemble_law_tiny_chisquare():
    """200 000 GPU samples of a 6-item L-ensemble against P(S) = det(C_S)/det(I + C)."""
    L = K = 6
    V = inputs.random_orthonormal(L, K, 106)
    lam = np.random.default_rng(106).uniform(0.05, 4.0, K)
    M = 200000
    gpos, gcnt, _ = run_gpu(V, lam, inputs.lens_uniforms(M, K, 11))
    subsets, p = exact.lensemble_set_probabilities(V, lam)
    index = {s: i for i, s in enumerate(subsets)}
    obs = np.bincount([index[tuple(sorted(r[:c]))] for r, c in zip(gpos.tolist(), gcnt.tolist())],
                      minlength=len(subsets))
    stat, dof, pval, _ = exact.pooled_chisquare(obs, p * M)
    assert pval > 1e-3, (stat, dof, pval)


def test_lensemble_full_workload():
    cfg = inputs.LENS
    V, lam = inputs.build_lensemble(cfg)
    uni = inputs.lens_uniforms(cfg.M, cfg.D, cfg.uniform_seed)
    gpos, gcnt, gfl = run_gpu(V, lam, uni)
    assert (gfl == 0).all()
    idx = np.unique(np.linspace(0, cfg.M - 1, 2000).round().astype(int))
    rpos, rcnt, _ = ref.sample_lensemble(V, lam, uni[idx])
    ex, ties = compare(V, lam, uni[idx], gpos[idx], gcnt[idx], rpos, rcnt)
    print(f"\nlens: {ex}/{len(idx)} spread samples bit-exact, {ties} CDF-boundary ties, mean N_i {gcnt.mean():.2f}")
    q = lam / (lam + 1)
    assert abs(gcnt.mean() - q.sum()) < 4 * np.sqrt((q * (1 - q)).sum() / cfg.M)
