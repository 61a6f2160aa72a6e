"""GPU modified-HKPV comparator (ffs_sample_hkpv) against the oracle (ref.sample_hkpv) on
identical seeded inputs: positions bit-exact except at CDF-boundary ties (|u - F| < 1e-9 on the
oracle's normalised CDF at the first divergent step, counted), several batches and ragged shapes,
real and complex, and the Eq. 1 law on a tiny system."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import exact, ref  # noqa: E402
from paper_2109_07358_b200 import inputs  # noqa: E402

pytestmark = pytest.mark.gpu
TIE_EPS = 1e-9


def _ffs():
    from paper_2109_07358_b200 import ffs
    return ffs


def run_gpu(U, uni):
    pos, fl = _ffs().ffs_sample_hkpv(torch.from_numpy(np.ascontiguousarray(U)).cuda(), torch.from_numpy(uni).cuda())
    torch.cuda.synchronize()
    return pos.cpu().numpy(), fl.cpu().numpy()


def compare(U, uni, gpos):
    rpos, rfl = ref.sample_hkpv(U, uni)
    ties = 0
    for i in np.nonzero((gpos != rpos).any(axis=1))[0]:
        k = int(np.argmax(gpos[i] != rpos[i]))
        _, _, w, _ = ref.sample_hkpv(U, uni[i:i + 1], S=1)
        F = np.cumsum(w[0, k])
        xs = int(rpos[i, k])
        lo = F[xs - 1] if xs > 0 else 0.0
        u = uni[i, k]
        assert abs(u - lo) < TIE_EPS or abs(u - F[xs]) < TIE_EPS, (i, k, gpos[i, k], xs, u, lo, F[xs])
        ties += 1
    return len(gpos) - ties, ties, rfl


SHAPES = [(16, 4, 4, False), (256, 32, 32, False), (300, 33, 20, False), (1024, 128, 128, False),
          (2100, 257, 40, False), (64, 21, 21, True), (500, 40, 40, True)]


@pytest.mark.parametrize("L,N,Np,cplx", SHAPES)
def test_hkpv_shapes_match_oracle(L, N, Np, cplx):
    U = inputs.random_orthonormal(L, N, 5 * L + N, complex_=cplx)
    M = 200 if L * N < 100000 else 60
    uni = np.random.Generator(np.random.Philox(L + N)).random((M, Np))
    gpos, gfl = run_gpu(U, uni)
    ex, ties, rfl = compare(U, uni, gpos)
    assert ex + ties == M
    assert (gfl == 0).all()
    assert all(len(set(p)) == Np for p in gpos.tolist())


def test_hkpv_batches(monkeypatch):
    """Several lockstep batches with a ragged last one (option dense_batch caps the batch)."""
    ffs = _ffs()
    ffs.set_option("dense_batch", 7)
    try:
        U = inputs.random_orthonormal(300, 20, 9)
        uni = np.random.Generator(np.random.Philox(10)).random((30, 20))
        gpos, _ = run_gpu(U, uni)
        ex, ties, _ = compare(U, uni, gpos)
        assert ex + ties == 30
    finally:
        ffs.reset_options()


def test_hkpv_tiny_law_chisquare():
    cfg = inputs.CONFIGS["tiny"]
    U = inputs.build_u(cfg)
    M = 200000
    gpos, _ = run_gpu(U, np.random.Generator(np.random.Philox(11)).random((M, cfg.N)))
    subsets, p = exact.set_probabilities(U)
    index = {s: i for i, s in enumerate(subsets)}
    obs = np.bincount([index[tuple(sorted(q))] for q in gpos.tolist()], minlength=len(subsets))
    stat, dof, pval, _ = exact.pooled_chisquare(obs, p * M)
    assert pval > 1e-3, (stat, dof, pval)


@pytest.mark.parametrize("L,N", [(16, 4), (256, 32), (100, 45)])
def test_hkpv_lockstep_path_at_small_L(L, N):
    """The lockstep GEMM path (option force_generic) on the shapes the warp kernel takes by default."""
    ffs = _ffs()
    ffs.set_option("force_generic", 1)
    try:
        U = inputs.random_orthonormal(L, N, 7 * L + N)
        uni = np.random.Generator(np.random.Philox(L)).random((150, N))
        gpos, gfl = run_gpu(U, uni)
        ex, ties, _ = compare(U, uni, gpos)
        assert ex + ties == 150 and (gfl == 0).all()
    finally:
        ffs.reset_options()
