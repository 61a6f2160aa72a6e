"""T0 — pins of the CPU oracle (oracle/) against what PAPER.md and the mathematics fix.

Every check compares the oracle with something other than itself: hand-derived values
(tests/golden), the Eq. 1 / Eq. 2 determinant definitions (numpy det), the Eq. 3 null-vector
definition (numpy SVD), closed forms of projection DPPs (K = U U^dagger), brute-force
enumeration and chi-square sampling tests. No GPU.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

from oracle import exact, ref
from paper_2109_07358_b200 import inputs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _rand_u(L, N, seed, cplx=False):
    return inputs.random_orthonormal(L, N, seed, complex_=cplx)


# ---------------------------------------------------------------- hand-derived worked example
def test_golden_worked_example():
    g = json.load(open(os.path.join(GOLDEN, "worked_example_l3n2.json")))
    U = np.array(g["U"])
    for c in g["cases"]:
        u = np.array(c["uniforms"])[None, :]
        m = ref.permutation(u[0, :2], 2)
        assert list(m) == c["m"]
        pos, w = ref.weights(U, u)
        assert list(pos[0]) == c["positions"]
        np.testing.assert_allclose(w[0], np.array(c["weights"]), atol=1e-15)
        _, hn2, tot = ref.chain(U, m, pos[0])
        np.testing.assert_allclose(hn2, c["hnorm2"], rtol=1e-14)
        np.testing.assert_allclose(tot, 1.0, rtol=1e-14)
        # chain determinant (Eq. 2 numerator): prod_k |u_{x_k}^T h'_k|^2 = |det U_{x,(m)}|^2
        prod = np.prod([w[0][k, pos[0][k]] * tot[k] * hn2[k] for k in range(2)])
        assert abs(prod - c["det2_chosen"]) < 1e-15


# ---------------------------------------------------------------- permutation rule (Q6)
def test_permutation_is_uniform_n4():
    from scipy import stats
    M = 48000
    u = inputs.uniforms(M, 4, 7)[:, :4]
    counts = {}
    for i in range(M):
        counts[tuple(ref.permutation(u[i], 4))] = counts.get(tuple(ref.permutation(u[i], 4)), 0) + 1
    assert len(counts) == 24
    obs = np.array(list(counts.values()))
    assert stats.chisquare(obs).pvalue > 1e-3


def test_partial_permutation_prefix_uniform():
    from scipy import stats
    M = 40000
    u = inputs.uniforms(M, 2, 8)[:, :2]
    counts = {}
    for i in range(M):
        k = tuple(ref.permutation(u[i], 5, 2)[:2])
        counts[k] = counts.get(k, 0) + 1
    assert len(counts) == 20  # all ordered pairs of 5 columns
    assert stats.chisquare(np.array(list(counts.values()))).pvalue > 1e-3


def test_identity_U_follows_permutation():
    # U = I (L = N): column m_k has its single nonzero at row m_k, so x_k = m_k exactly.
    N = 6
    U = np.eye(N)
    uni = inputs.uniforms(200, N, 3)
    pos = ref.sample(U, uni)
    for i in range(200):
        assert list(pos[i]) == list(ref.permutation(uni[i, :N], N))


# ---------------------------------------------------------------- selection rule (Q5)
def test_selection_rule_strict_index_order():
    U = np.full((4, 1), 0.5)  # w = 0.25 each, exactly; T = 1 exactly
    for us, want in [(0.0, 0), (0.2499999, 0), (0.25, 1), (0.5, 2), (0.74999, 2), (0.75, 3),
                     (0.9999999999999999, 3)]:
        pos = ref.sample(U, np.array([[0.3, us]]))
        assert pos[0, 0] == want, (us, pos)


# ---------------------------------------------------------------- conditionals vs definitions
@pytest.mark.parametrize("cplx", [False, True])
def test_conditional_equals_determinant_ratio(cplx):
    rng = np.random.default_rng(11)
    for trial in range(6):
        L, N = 7, 4
        U = _rand_u(L, N, 100 + trial, cplx)
        m = rng.permutation(N).astype(np.int32)
        x = rng.choice(L, N, replace=False).astype(np.int32)
        w, _, _ = ref.chain(U, m, x)
        for k in range(N):
            want = exact.det_conditional(U, m, list(x[:k]))
            np.testing.assert_allclose(w[k], want, atol=1e-13, rtol=0)


@pytest.mark.parametrize("cplx", [False, True])
def test_conditional_equals_nullvector_definition(cplx):
    L, N = 64, 16
    U = _rand_u(L, N, 5, cplx)
    uni = inputs.uniforms(3, N, 21)
    pos, w = ref.weights(U, uni)
    for i in range(3):
        m = ref.permutation(uni[i, :N], N)
        for k in range(N):
            want = exact.nullvec_conditional(U, m, list(pos[i, :k]))
            assert np.max(np.abs(w[i, k] - want)) <= 1e-12 * np.max(want)


@pytest.mark.parametrize("cplx", [False, True])
def test_mixture_identity_eq2(cplx):
    # Eq. 2: sum_m prod_k P(x_k | x_<k; m) = |det U_{x,n}|^2 for every ordered x.
    L, N = 5, 3
    U = _rand_u(L, N, 17, cplx)
    perms = [np.array(p, dtype=np.int32) for p in itertools.permutations(range(N))]
    worst = 0.0
    for x in itertools.permutations(range(L), N):
        x = np.array(x, dtype=np.int32)
        s = 0.0
        for m in perms:
            w, _, _ = ref.chain(U, m, x)
            s += np.prod([w[k, x[k]] for k in range(N)])
        worst = max(worst, abs(s - abs(np.linalg.det(U[x, :])) ** 2))
    assert worst < 1e-13


def test_k1_weights_are_column_moduli():
    U = _rand_u(20, 5, 2, True)
    m = np.array([3, 1, 4, 0, 2], dtype=np.int32)
    w, _, _ = ref.chain(U, m, np.array([0], dtype=np.int32))
    np.testing.assert_allclose(w[0], np.abs(U[:, 3]) ** 2, atol=1e-15)


@pytest.mark.parametrize("cplx", [False, True])
def test_normalisation_and_chain_determinant(cplx):
    # U^dagger U = 1 => sum_x |u_x^T h|^2 = |h|^2 = 1 (unit h); prod_k |u_{x_k}^T h'_k|^2 = |det V_{X,1..N}|^2
    L, N = 32, 8
    U = _rand_u(L, N, 23, cplx)
    uni = inputs.uniforms(5, N, 4)
    pos, w = ref.weights(U, uni)
    for i in range(5):
        m = ref.permutation(uni[i, :N], N)
        wc, hn2, tot = ref.chain(U, m, pos[i])
        np.testing.assert_allclose(tot, 1.0, atol=1e-13)
        np.testing.assert_allclose(w[i].sum(axis=1), 1.0, atol=1e-13)
        prod = np.prod([wc[k, pos[i, k]] * tot[k] * hn2[k] for k in range(N)])
        det2 = abs(np.linalg.det(U[np.ix_(pos[i], m)])) ** 2
        assert abs(prod - det2) <= 1e-10 * det2


# ---------------------------------------------------------------- special cases
def test_point_mass():
    U = np.zeros((5, 1))
    U[2, 0] = 1.0
    pos = ref.sample(U, inputs.uniforms(100, 1, 5))
    assert (pos[:, 0] == 2).all()


@pytest.mark.parametrize("cplx", [False, True])
def test_full_filling(cplx):
    U = _rand_u(3, 3, 9, cplx)
    pos = ref.sample(U, inputs.uniforms(500, 3, 6))
    assert all(sorted(p) == [0, 1, 2] for p in pos.tolist())


def test_pauli_exclusion_and_range():
    U = _rand_u(40, 12, 1)
    pos = ref.sample(U, inputs.uniforms(2000, 12, 2))
    assert pos.min() >= 0 and pos.max() < 40
    assert all(len(set(p)) == 12 for p in pos.tolist())


def test_marginal_np_equal_n_is_full():
    U = _rand_u(30, 6, 12)
    uni = inputs.uniforms(300, 6, 13)
    a = ref.sample(U, uni)
    b = ref.sample(U, uni, Np=6)
    assert (a == b).all()


# ---------------------------------------------------------------- output law (Eq. 1)
def test_chisquare_tiny_config_against_bruteforce():
    # BASELINE configs[0]: L=16, N=4, M=200000; histogram vs |det U_S|^2 over all 1820 sets.
    cfg = inputs.CONFIGS["tiny"]
    U = inputs.build_u(cfg)
    subsets, p = exact.set_probabilities(U)
    assert abs(p.sum() - 1.0) < 1e-13  # Cauchy-Binet
    pos = ref.sample(U, inputs.uniforms(cfg.M, cfg.N, cfg.uniform_seed))
    index = {s: i for i, s in enumerate(subsets)}
    obs = np.bincount([index[tuple(sorted(r))] for r in pos.tolist()], minlength=len(subsets))
    stat, dof, pval, nb = exact.pooled_chisquare(obs, p * cfg.M)
    assert pval > 1e-3, (stat, dof, pval)
    # (TV over 1820 bins at M=2e5 has a sampling floor of ~0.02, so only the chi-square is asserted)


def test_chisquare_complex_small():
    U = _rand_u(6, 3, 31, True)
    subsets, p = exact.set_probabilities(U)
    M = 60000
    pos = ref.sample(U, inputs.uniforms(M, 3, 32))
    index = {s: i for i, s in enumerate(subsets)}
    obs = np.bincount([index[tuple(sorted(r))] for r in pos.tolist()], minlength=len(subsets))
    assert exact.pooled_chisquare(obs, p * M)[2] > 1e-3


# ---------------------------------------------------------------- marginal
@pytest.mark.parametrize("cplx", [False, True])
def test_marginal_exact_enumeration(cplx):
    # E_m[P(x_1|m) P(x_2|x_1;m)] over all N! permutations equals det K[x,x] (N-N')!/N!.
    L, N, Np = 6, 3, 2
    U = _rand_u(L, N, 41, cplx)
    perms = [np.array(p, dtype=np.int32) for p in itertools.permutations(range(N))]
    for xs in itertools.permutations(range(L), Np):
        xs = np.array(xs, dtype=np.int32)
        s = 0.0
        for m in perms:
            w, _, _ = ref.chain(U, m, xs)
            s += w[0, xs[0]] * w[1, xs[1]]
        s /= math.factorial(N)
        assert abs(s - exact.ordered_marginal_probability(U, xs)) < 1e-14


def test_marginal_sampling_chisquare():
    L, N, Np = 6, 3, 2
    U = _rand_u(L, N, 43)
    M = 60000
    pos = ref.sample(U, inputs.uniforms(M, Np, 44), Np=Np)
    pairs = list(itertools.permutations(range(L), Np))
    expected = np.array([exact.ordered_marginal_probability(U, q) for q in pairs]) * M
    idx = {q: i for i, q in enumerate(pairs)}
    obs = np.bincount([idx[tuple(r)] for r in pos.tolist()], minlength=len(pairs))
    assert abs(expected.sum() - M) < 1e-6 * M
    assert exact.pooled_chisquare(obs, expected)[2] > 1e-3


def test_marginal_one_step_is_kxx_over_n():
    U = _rand_u(12, 4, 45)
    M = 80000
    pos = ref.sample(U, inputs.uniforms(M, 1, 46), Np=1)
    K = np.sum(np.abs(U) ** 2, axis=1)
    from scipy import stats
    obs = np.bincount(pos[:, 0], minlength=12)
    assert stats.chisquare(obs, K / 4 * M).pvalue > 1e-3


# ---------------------------------------------------------------- mid-size config: occupations
def test_occupation_double_well_config():
    # <n_x> = K_xx (projection DPP), z-test with Bonferroni over sites.
    cfg = inputs.CONFIGS["dw"]
    U = inputs.build_u(cfg)
    M = 8000
    pos = ref.sample(U, inputs.uniforms(M, cfg.N, cfg.uniform_seed)[:M])
    occ = np.bincount(pos.ravel(), minlength=cfg.L) / M
    K = np.sum(U ** 2, axis=1)
    se = np.sqrt(np.maximum(K * (1 - K), 1e-12) / M)
    z = np.abs(occ - K) / se
    assert z.max() < 4.5
    assert abs(occ.sum() - cfg.N) < 1e-9


# ---------------------------------------------------------------- argument handling
def test_bad_arguments_rejected():
    L = ref.lib()
    U = np.zeros((4, 2))
    uni = np.zeros((1, 4))
    pos = np.zeros((1, 2), dtype=np.int32)
    assert L.ffs_ref_sample_marginal(U.ctypes.data, 4, 5, 0, 1, 2, uni.ctypes.data, pos.ctypes.data, None, 1) == -1
    assert L.ffs_ref_sample_marginal(U.ctypes.data, 4, 2, 0, 1, 3, uni.ctypes.data, pos.ctypes.data, None, 1) == -1
    assert L.ffs_ref_sample_marginal(U.ctypes.data, 4, 2, 7, 1, 2, uni.ctypes.data, pos.ctypes.data, None, 1) == -1
    assert L.ffs_ref_sample_marginal(U.ctypes.data, 4, 2, 0, 0, 2, None, None, None, 1) == 0


# ---------------------------------------------------------------- L-ensemble front end
def _lens_inputs(L, K, seed, cplx=False):
    V = _rand_u(L, K, seed, cplx)
    lam = np.random.default_rng(seed).uniform(0.05, 4.0, K)
    return V, lam


def _lens_uniforms(M, K, seed):
    return np.random.Generator(np.random.Philox(seed)).random((M, 3 * K))


@pytest.mark.parametrize("L,K,cplx", [(6, 6, False), (7, 4, False), (5, 5, True)])
def test_lensemble_matches_brute_force_law(L, K, cplx):
    """Sampled subsets follow P(S) = det(C_S)/det(I + C), C = V diag(lam) V^dagger: the L-ensemble
    the paper's pipeline samples by keeping eigenvector j w.p. lam_j/(lam_j+1) and running FFS."""
    V, lam = _lens_inputs(L, K, 100 + L + K, cplx)
    M = 200000
    pos, cnt, flags = ref.sample_lensemble(V, lam, _lens_uniforms(M, K, 5 + L))
    assert (flags == 0).all()
    assert (cnt <= K).all() and (pos[np.arange(K)[None, :] >= cnt[:, None]] == -1).all()
    subsets, p = exact.lensemble_set_probabilities(V, lam)
    assert abs(p.sum() - 1.0) < 1e-12  # normalisation of the definition
    index = {s: i for i, s in enumerate(subsets)}
    obs = np.bincount([index[tuple(sorted(r[:c]))] for r, c in zip(pos.tolist(), cnt.tolist())],
                      minlength=len(subsets))
    stat, dof, pval, _ = exact.pooled_chisquare(obs, p * M)
    assert pval > 1e-3, (stat, dof, pval)


def test_lensemble_size_distribution():
    """N_i is a sum of independent Bernoulli(lam_j/(lam_j+1)): mean and variance."""
    L, K = 40, 24
    V, lam = _lens_inputs(L, K, 3)
    M = 20000
    _, cnt, _ = ref.sample_lensemble(V, lam, _lens_uniforms(M, K, 9))
    q = lam / (lam + 1)
    mu, var = q.sum(), (q * (1 - q)).sum()
    assert abs(cnt.mean() - mu) < 4 * np.sqrt(var / M)
    assert abs(cnt.var() / var - 1) < 0.1


def test_lensemble_degenerate_spectra():
    """lam = 0 keeps nothing (empty sample); lam -> inf keeps every eigenvector, and the sample is
    then plain FFS of V driven by the permutation / selection blocks of the same uniform row."""
    L, K = 12, 5
    V = _rand_u(L, K, 21)
    uni = _lens_uniforms(300, K, 4)
    pos, cnt, _ = ref.sample_lensemble(V, np.zeros(K), uni)
    assert (cnt == 0).all() and (pos == -1).all()
    pos, cnt, _ = ref.sample_lensemble(V, np.full(K, 1e300), uni)
    assert (cnt == K).all()
    assert (pos == ref.sample(V, uni[:, K:])).all()


# ---------------------------------------------------------------- observables and reweighting (Supp S5)
def test_occupation_and_pair_closed_forms():
    """Projection DPP identities (K = U U^dagger): <n_x> = K_xx and <n_x n_y> = K_xx K_yy - |K_xy|^2
    (z-tests), the sum rule sum_x n_x = N per sample (exact), diagonal pair counts = occupations."""
    L, N, M = 12, 4, 100000
    U = _rand_u(L, N, 31)
    pos = ref.sample(U, inputs.uniforms(M, N, 32))
    occ = ref.occupation(pos, L)
    assert int(occ.sum()) == M * N
    K = U @ U.conj().T
    kxx = np.real(np.diag(K))
    z = (occ / M - kxx) / np.sqrt(kxx * (1 - kxx) / M)
    assert np.abs(z).max() < 4.5
    pair = ref.pair_occupation(pos, L)
    assert (np.diag(pair) == occ).all() and (pair == pair.T).all()
    assert (pair.sum(axis=1) == N * occ).all()
    g = np.outer(kxx, kxx) - np.abs(K) ** 2
    np.fill_diagonal(g, kxx)
    zp = (pair / M - g) / np.sqrt(np.maximum(g * (1 - g), 1e-12) / M)
    assert np.abs(zp).max() < 5.0


def test_gutzwiller_reweighting_matches_enumeration():
    """<O>_J = <J^2 O>_0/<J^2>_0 from free FFS samples equals the exact interacting expectation of
    the Gutzwiller-projected state (enumeration over all spinful configurations), within 4.5 sigma
    of the ratio estimator."""
    L, N, V, Ms = 5, 2, 1.5, 100000
    U = _rand_u(L, N, 41)
    pos = ref.sample(U, inputs.uniforms(2 * Ms, N, 42))
    res = ref.gutzwiller(pos, L, V)
    ex = exact.gutzwiller_exact(U, V)
    w = ex["p0"] * ex["J2"] / ex["J2_0"]

    def se(o, mean):  # delta-method s.e. of sum J2 O / sum J2 under P_0
        return np.sqrt(np.sum(ex["p0"] * (ex["J2"] / ex["J2_0"]) ** 2 * (o - mean) ** 2) / Ms)

    assert abs(res[0] - ex["J2_0"]) < 4.5 * np.sqrt(np.sum(ex["p0"] * (ex["J2"] - ex["J2_0"]) ** 2) / Ms)
    assert abs(res[1] - ex["D_J"]) < 4.5 * se(ex["D"], ex["D_J"])
    for x in range(L):
        assert abs(res[2 + x] - ex["n_J"][x]) < 4.5 * se(ex["n"][:, x], ex["n_J"][x])
    # the reweighting moves the estimate: <D>_J < <D>_0 for V > 0
    assert ex["D_J"] < np.sum(ex["p0"] * ex["D"]) - 0.05
    assert abs(w.sum() - 1) < 1e-12


def test_gutzwiller_special_cases():
    """V = 0: unit weights, <n_x>_J is the plain sample mean (both spins), <J^2>_0 = 1; a
    hand-built pair set with known double occupancies gives the closed-form weighted mean."""
    L, N = 10, 3
    U = _rand_u(L, N, 51)
    pos = ref.sample(U, inputs.uniforms(400, N, 52))
    r0 = ref.gutzwiller(pos, L, 0.0)
    assert r0[0] == 1.0
    np.testing.assert_allclose(r0[2:], ref.occupation(pos, L) / 200.0, rtol=0, atol=1e-14)
    # two spinful samples: D = 2 (x = 0, 1 doubly occupied) and D = 0
    pos = np.array([[0, 1, 2], [1, 0, 5], [3, 4, 6], [7, 8, 9]], dtype=np.int32)
    V = 0.7
    r = ref.gutzwiller(pos, L, V)
    w1, w2 = np.exp(-2 * V), 1.0
    assert abs(r[0] - (w1 + w2) / 2) < 1e-15
    assert abs(r[1] - 2 * w1 / (w1 + w2)) < 1e-15
    n = np.zeros(L)
    n[[0, 1]] = 2 * w1
    n[[2, 5]] = w1
    n[[3, 4, 6, 7, 8, 9]] = w2
    np.testing.assert_allclose(r[2:], n / (w1 + w2), rtol=1e-15)


# ---------------------------------------------------------------- Supp S7 Metropolis variant
def _metro_uniforms(M, Np, Mc, seed):
    return np.random.Generator(np.random.Philox(seed)).random((M, Np + Np * (1 + 2 * Mc)))


def test_metropolis_without_updates_keeps_the_initial_draw():
    """M_cond = 0: x_k is the chain's start floor(u_init L) (PAPER.md:388 with no iteration)."""
    L, N = 30, 3
    U = _rand_u(L, N, 61)
    uni = _metro_uniforms(500, N, 0, 62)
    pos, flags = ref.sample_metropolis(U, uni, N, 0)
    starts = np.floor(uni[:, N:] * L).astype(int)
    assert (pos == starts).all()


def test_metropolis_accept_rule():
    """u_acc = 0 accepts every proposal with positive weight (0 * w(x) < w(x')), so the chain ends
    on the last proposal that is not an already chosen site (those have weight 0, Pauli)."""
    L, N, Mc = 25, 4, 6
    U = _rand_u(L, N, 63)
    uni = _metro_uniforms(300, N, Mc, 64)
    for k in range(N):
        uni[:, N + k * (1 + 2 * Mc) + 2:N + (k + 1) * (1 + 2 * Mc):2] = 0.0
    pos, flags = ref.sample_metropolis(U, uni, N, Mc)
    for i in range(300):
        chosen = set()
        for k in range(N):
            c = uni[i, N + k * (1 + 2 * Mc):N + (k + 1) * (1 + 2 * Mc)]
            x = int(np.floor(c[0] * L))
            for t in range(Mc):
                xp = int(np.floor(c[1 + 2 * t] * L))
                if xp not in chosen:
                    x = xp
            assert pos[i, k] == x
            chosen.add(x)


def test_metropolis_single_particle_stationary_law():
    """N = 1: the chain targets w(x) = |U[x,0]|^2 (Eq. 3 with k = 1); after Mc = 100 independent
    uniform proposals the draws follow it (chi-square), as the paper's N = 1 continuous example."""
    from scipy import stats
    L, M = 20, 100000
    U = _rand_u(L, 1, 65)
    pos, _ = ref.sample_metropolis(U, _metro_uniforms(M, 1, 100, 66), 1, 100)
    p = np.abs(U[:, 0]) ** 2
    obs = np.bincount(pos[:, 0], minlength=L)
    assert stats.chisquare(obs, p * M).pvalue > 1e-3


@pytest.mark.parametrize("cplx", [False, True])
def test_metropolis_tiny_law(cplx):
    """SPEC.md:193 acceptance example: L = 6, N = 2, M_cond = 500 discrete updates -> the sampled
    sets follow |det U_S|^2 (Eq. 1): chi-square and TV <= 0.02 (100 000 samples)."""
    L, N, M, Mc = 6, 2, 100000, 200
    U = _rand_u(L, N, 67, cplx)
    pos, flags = ref.sample_metropolis(U, _metro_uniforms(M, N, Mc, 68), N, Mc)
    assert (flags == 0).all()
    subsets, p = exact.set_probabilities(U)
    index = {s: i for i, s in enumerate(subsets)}
    obs = np.bincount([index[tuple(sorted(q))] for q in pos.tolist()], minlength=len(subsets))
    stat, dof, pval, _ = exact.pooled_chisquare(obs, p * M)
    assert pval > 1e-3, (stat, dof, pval)
    assert 0.5 * np.abs(obs / M - p).sum() <= 0.02


# ---------------------------------------------------------------- modified HKPV comparator
@pytest.mark.parametrize("cplx", [False, True])
def test_hkpv_conditionals_are_schur_complements_of_K(cplx):
    """The HKPV chain rule on K = U U^dagger: the step-k weight of x is the Schur complement
    K_xx - K_{x,X} K_XX^{-1} K_{X,x} of the chosen set X (normalised by its trace N - k + 1),
    and the totals obey the trace identity sum_x r_k(x) = N - (k-1)."""
    L, N = 11, 5
    U = _rand_u(L, N, 71, cplx)
    uni = np.random.Generator(np.random.Philox(72)).random((6, N))
    pos, _, w, tot = ref.sample_hkpv(U, uni, S=6)
    K = U @ U.conj().T
    for i in range(6):
        for k in range(N):
            X = list(pos[i, :k])
            r = np.real(np.diag(K)).copy()
            if X:
                KX = K[np.ix_(range(L), X)]
                r -= np.real(np.einsum("xa,ab,xb->x", KX, np.linalg.inv(K[np.ix_(X, X)]), KX.conj()))
                r[X] = 0.0
            np.testing.assert_allclose(w[i, k], np.maximum(r, 0) / (N - k), atol=1e-12)
            assert abs(tot[i, k] - (N - k)) < 1e-12


@pytest.mark.parametrize("L,N,cplx", [(6, 3, False), (16, 4, False), (5, 2, True)])
def test_hkpv_matches_brute_force_law(L, N, cplx):
    U = _rand_u(L, N, 73 + L, cplx) if (L, N) != (16, 4) else inputs.build_u(inputs.CONFIGS["tiny"])
    M = 200000
    pos, flags = ref.sample_hkpv(U, np.random.Generator(np.random.Philox(74)).random((M, N)))
    assert (flags == 0).all()
    subsets, p = exact.set_probabilities(U)
    index = {s: i for i, s in enumerate(subsets)}
    obs = np.bincount([index[tuple(sorted(q))] for q in pos.tolist()], minlength=len(subsets))
    stat, dof, pval, _ = exact.pooled_chisquare(obs, p * M)
    assert pval > 1e-3, (stat, dof, pval)


def test_hkpv_special_cases():
    """Point mass (U = e_3 column), full filling (L = N), first step K_xx / N."""
    U = np.zeros((5, 1))
    U[2, 0] = 1.0
    pos, _ = ref.sample_hkpv(U, np.random.default_rng(1).random((50, 1)))
    assert (pos == 2).all()
    U = _rand_u(4, 4, 75)
    pos, _ = ref.sample_hkpv(U, np.random.default_rng(2).random((50, 4)))
    assert all(sorted(p) == [0, 1, 2, 3] for p in pos.tolist())
    U = _rand_u(9, 3, 76)
    _, _, w, _ = ref.sample_hkpv(U, np.random.default_rng(3).random((1, 3)), S=1)
    np.testing.assert_allclose(w[0, 0], np.sum(U ** 2, axis=1) / 3, atol=1e-15)


# ---------------------------------------------------------------- oracle vs definition at full scale
@pytest.mark.parametrize("name,steps", [("anderson", (1, 17, 64, 128)), ("peierls", (1, 40, 200)),
                                        ("dpp", (1, 64, 257))])
def test_oracle_matches_definition_at_scale(name, steps):
    """the oracle's eager-elimination conditionals vs the Eq. 3 definition (numpy SVD
    null vector of the chosen rows, then |u_x^T h|^2 over all L candidates) on 2 samples of the C3,
    C4 and C5 configurations, at a subset of steps along the oracle's own path; normwise <= 1e-12
    (the survey's measured floor between two correct fp64 methods is 1.5e-11 only at k = N = 1024,
    SURVEY App. A; these steps stay below it)."""
    cfg = inputs.CONFIGS[name]
    U = inputs.build_u(cfg)
    kmax = max(steps)
    uni = inputs.uniforms(2, kmax, cfg.uniform_seed + 7)
    pos = ref.sample(U, uni, Np=kmax)
    for s in range(2):
        m = ref.permutation(uni[s, :kmax], cfg.N, kmax)
        w, _, _ = ref.chain(U, m, pos[s])
        for k in steps:
            wd = exact.nullvec_conditional(U, m, list(pos[s, :k - 1]))
            err = np.max(np.abs(w[k - 1] - wd)) / np.max(wd)
            assert err <= 1e-12, (name, s, k, err)
