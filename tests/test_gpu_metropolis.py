"""Supp S7 Metropolis variant on the GPU (ffs_sample_metropolis) against the oracle
(ref.sample_metropolis) on identical seeded inputs: positions bit-exact except where an
accept/reject decision of the oracle's chain lies within 1e-9 of flipping (|u_acc - w'/w| < 1e-9,
the analogue of the CDF-boundary tie; counted), the Eq. 1 law on a tiny system, and the full-size
continuous-model stand-in (L = 2^20 grid) on spread samples."""
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


def run_gpu(U, uni, Np, Mc):
    pos, flags = _ffs().ffs_sample_metropolis(torch.from_numpy(np.ascontiguousarray(U)).cuda(),
                                              torch.from_numpy(uni).cuda(), Np, Mc)
    torch.cuda.synchronize()
    return pos.cpu().numpy(), flags.cpu().numpy()


def compare(U, uni, Np, Mc, gpos):
    rpos, rfl, mg = ref.sample_metropolis(U, uni, Np, Mc, return_margins=True)
    ties = 0
    for i in np.nonzero((gpos != rpos).any(axis=1))[0]:
        k = int(np.argmax(gpos[i] != rpos[i]))
        assert mg[i, k] < TIE_EPS, (i, k, gpos[i, k], rpos[i, k], mg[i, k])
        ties += 1
    return len(gpos) - ties, ties, rfl


SHAPES = [  # (L, N, N', Mc, complex)
    (30, 6, 6, 0, False), (30, 6, 6, 1, False), (200, 20, 13, 7, False), (1000, 40, 40, 33, False),
    (5000, 64, 20, 40, False), (3000, 100, 100, 5, False), (100000, 16, 16, 64, False),
    (64, 10, 10, 9, True), (2000, 30, 17, 32, True),
]


@pytest.mark.parametrize("L,N,Np,Mc,cplx", SHAPES)
def test_metropolis_shapes_match_oracle(L, N, Np, Mc, cplx):
    U = inputs.random_orthonormal(L, N, L + N + Mc, complex_=cplx) if L <= 5000 else inputs.build_box_orbitals(L, N)
    M = 300
    uni = inputs.metro_uniforms(M, Np, Mc, 3 * L + Mc)
    gpos, gfl = run_gpu(U, uni, Np, Mc)
    ex, ties, rfl = compare(U, uni, Np, Mc, gpos)
    assert ex + ties == M
    assert (gfl == rfl).all()
    # Pauli exclusion wherever the chains ended on positive weight (bit2 flags a too-short chain
    # that stayed on a zero-weight, e.g. already chosen, start)
    assert all(len(set(p)) == Np for p, f in zip(gpos.tolist(), gfl.tolist()) if not f & 4)


def test_metropolis_tiny_law_chisquare():
    L, N, M, Mc = 6, 2, 200000, 200
    U = inputs.random_orthonormal(L, N, 67)
    gpos, gfl = run_gpu(U, inputs.metro_uniforms(M, N, Mc, 5), N, Mc)
    assert (gfl == 0).all()
    subsets, p = exact.set_probabilities(U)
    index = {s: i for i, s in enumerate(subsets)}
    obs = np.bincount([index[tuple(sorted(q))] for q in gpos.tolist()], minlength=len(subsets))
    stat, dof, pval, _ = exact.pooled_chisquare(obs, p * M)
    assert pval > 1e-3, (stat, dof, pval)


def test_metropolis_full_workload():
    cfg = inputs.METRO
    U = inputs.build_box_orbitals(cfg.L, cfg.N)
    uni = inputs.metro_uniforms(cfg.M, cfg.N, cfg.Mc, cfg.uniform_seed)
    gpos, gfl = run_gpu(U, uni, cfg.N, cfg.Mc)
    assert (gfl == 0).all()
    assert gpos.min() >= 0 and gpos.max() < cfg.L
    assert (np.diff(np.sort(gpos, axis=1), axis=1) > 0).all()
    idx = np.unique(np.linspace(0, cfg.M - 1, 64).round().astype(int))
    ex, ties, _ = compare(U, uni[idx], cfg.N, cfg.Mc, gpos[idx])
    print(f"\nmetro: {ex}/{len(idx)} spread samples bit-exact, {ties} decision ties")
