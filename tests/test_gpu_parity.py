"""T1/T2 — the CUDA path (through the C ABI) against the oracle on identical seeded inputs.

Small shapes cover every kernel variant (warp owners with shared/global U^T, CTA owners of each
register-capacity class, real and complex), several panel blocks and ragged tails (L not a
multiple of the owner's rows, N' not a multiple of the panel width). Full BASELINE.json sizes
run in the launch configuration bench.py times, compared on a prefix of samples the oracle
finishes in seconds, plus properties that hold at any size (occupations = K_xx).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import exact, ref  # noqa: E402
from paper_2109_07358_b200 import inputs  # noqa: E402
from tests.parity import WEIGHT_TOL, compare_positions, compare_weights  # noqa: E402

pytestmark = pytest.mark.gpu


def _ffs():
    from paper_2109_07358_b200 import ffs
    return ffs


def _to_dev(U):
    return torch.from_numpy(np.ascontiguousarray(U)).cuda()


@pytest.fixture(autouse=True)
def _default_options():
    """Every test starts and ends with the library's default tuning options."""
    if torch.cuda.is_available():
        _ffs().reset_options()
    yield
    if torch.cuda.is_available():
        _ffs().reset_options()


def run_gpu(U, uni, Np, trace_S=0, trace_S0=0):
    ffs = _ffs()
    Ud = _to_dev(U)
    ud = torch.from_numpy(uni).cuda()
    if trace_S:
        pos, flags, w = ffs.ffs_debug_trace(Ud, ud, Np, trace_S, S0=trace_S0)
        torch.cuda.synchronize()
        return pos.cpu().numpy(), flags.cpu().numpy(), w.cpu().numpy()
    if Np == U.shape[1]:
        pos, flags = ffs.ffs_sample(Ud, ud, with_flags=True)
    else:
        pos, flags = ffs.ffs_sample_marginal(Ud, ud, Np, with_flags=True)
    torch.cuda.synchronize()
    return pos.cpu().numpy(), flags.cpu().numpy(), None


SMALL = [
    # (L, N, N', complex) — spans every variant of pick_variant() and ragged tails
    (16, 4, 4, False), (7, 3, 3, False), (32, 9, 9, False), (50, 17, 17, False),
    (100, 23, 23, False), (128, 40, 13, False), (256, 32, 32, False), (200, 60, 60, False),
    (256, 90, 90, False), (300, 33, 33, False),
    (129, 9, 9, False), (160, 45, 45, False), (250, 48, 17, False), (256, 5, 5, False),
    (2048, 256, 256, False), (3000, 260, 260, False), (1024, 40, 21, False), (1500, 19, 19, False),
    (5000, 11, 11, False), (9000, 7, 7, False),
    (16, 4, 4, True), (30, 11, 11, True), (64, 21, 9, True), (128, 30, 30, True),
    (500, 26, 26, True), (2000, 9, 9, True), (6000, 5, 5, True), (2048, 256, 256, True), (2500, 258, 258, True),
]


@pytest.mark.parametrize("L,N,Np,cplx", SMALL)
def test_small_shapes_match_oracle(L, N, Np, cplx):
    U = inputs.random_orthonormal(L, N, 1000 + L + N, complex_=cplx)
    M = 300 if L * N < 200000 else 60
    uni = inputs.uniforms(M, Np, L * 7 + N)
    gpos, gflags, gw = run_gpu(U, uni, Np, trace_S=3)
    rpos, rflags = ref.sample(U, uni, Np=Np, return_flags=True)
    r = compare_positions(U, uni, gpos, rpos, Np)
    assert not r["failures"], r
    assert r["exact"] + r["ties"] == M
    assert (gflags == 0).all()
    # Pauli exclusion / range
    assert all(len(set(p)) == Np for p in gpos.tolist())
    _, rw = ref.weights(U, uni[:3], Np=Np)
    assert compare_weights(gw, rw, gpos, rpos) <= WEIGHT_TOL


def test_tiny_config_full_M_bitexact_and_chisquare():
    cfg = inputs.CONFIGS["tiny"]
    U = inputs.build_u(cfg)
    uni = inputs.uniforms(cfg.M, cfg.N, cfg.uniform_seed)
    gpos, gflags, _ = run_gpu(U, uni, cfg.N)
    rpos = ref.sample(U, uni)
    r = compare_positions(U, uni, gpos, rpos, cfg.N)
    assert not r["failures"], r["failures"][:5]
    subsets, p = exact.set_probabilities(U)
    index = {s: i for i, s in enumerate(subsets)}
    obs = np.bincount([index[tuple(sorted(q))] for q in gpos.tolist()], minlength=len(subsets))
    stat, dof, pval, _ = exact.pooled_chisquare(obs, p * cfg.M)
    assert pval > 1e-3, (stat, dof, pval)


# (config, N', oracle sample indices, traced samples): the compared samples are spread over the
# whole run (first / middle / last tiles, clusters and lockstep batches), and the traced samples
# are the LAST ones of the full-size launch (ffs_debug_trace S0), so the weights are checked in
# the last tiles too. Sizes: what the oracle on the GPU box's host cores finishes in ~1 minute.
def _spread(M, n):
    return sorted(set(np.linspace(0, M - 1, n).round().astype(int).tolist()))


FULL = [
    ("dw", None, 3000, 4),
    ("anderson", None, 300, 2),
    ("anderson", 16, 4000, 8),
    ("peierls", None, 24, 2),
    ("dpp", None, 8, 1),
    ("dpp", 64, 400, 4),
]

FULL_WEIGHT_TOL = 1e-11  # 10x inside the 1e-10 bound: emulation or blocking drift shows before parity breaks


@pytest.mark.parametrize("name,Np,n_ref,n_trace", FULL)
def test_full_size_configs(name, Np, n_ref, n_trace):
    cfg = inputs.CONFIGS[name]
    U = inputs.build_u(cfg)
    Np = cfg.N if Np is None else Np
    M = cfg.M if Np == cfg.N else cfg.marginal_M
    uni = inputs.uniforms(M, Np, cfg.uniform_seed + (0 if Np == cfg.N else 100))
    gpos, gflags, tw = run_gpu(U, uni, Np, trace_S=n_trace, trace_S0=M - n_trace)
    assert (gflags == 0).all()
    assert gpos.min() >= 0 and gpos.max() < cfg.L
    srt = np.sort(gpos, axis=1)
    assert (np.diff(srt, axis=1) > 0).all()  # Pauli exclusion, every sample
    idx = np.array(_spread(M, n_ref))
    rpos = ref.sample(U, uni[idx], Np=Np)
    r = compare_positions(U, uni[idx], gpos[idx], rpos, Np)
    print(f"\n{name} N'={Np}: {r['exact']}/{len(idx)} compared samples bit-exact "
          f"(indices {idx[0]}..{idx[-1]}), {r['ties']} CDF-boundary ties")
    assert not r["failures"], r["failures"][:5]
    # weights along the path of the last n_trace samples of the full-size launch
    last = np.arange(M - n_trace, M)
    rlast, rw = ref.weights(U, uni[last], Np=Np)
    err = compare_weights(tw, rw, gpos[last], rlast)
    print(f"{name} N'={Np}: max normwise weight error {err:.3e} over samples {last[0]}..{last[-1]}")
    assert err <= FULL_WEIGHT_TOL
    # property at full size: occupation of each site = K_xx * N'/N (exchangeable order)
    K = np.sum(np.abs(U) ** 2, axis=1) * (Np / cfg.N)
    check_occupations(gpos, K, M)


def check_occupations(pos, K, M):
    """<n_x> = K_xx N'/N: z-test (Bonferroni) where M K(1-K) >= 10; the sites with few expected
    counts are pooled and checked against the Poisson tail."""
    from scipy import stats
    occ = np.bincount(pos.ravel(), minlength=K.shape[0])
    big = M * K * (1 - K) >= 10
    z = np.abs(occ[big] / M - K[big]) / np.sqrt(K[big] * (1 - K[big]) / M)
    assert z.max() < stats.norm.isf(1e-3 / (2 * max(1, big.sum()))), (z.max(), np.nonzero(big)[0][np.argmax(z)])
    lam = M * K[~big].sum()
    obs = occ[~big].sum()
    if lam > 0:
        assert stats.poisson.sf(obs - 1, lam) > 1e-4 and stats.poisson.cdf(obs, lam) > 1e-4, (obs, lam)


def test_edge_cases():
    ffs = _ffs()
    L = ffs.load()
    U = inputs.random_orthonormal(10, 3, 5)
    Ud = _to_dev(U)
    ud = torch.from_numpy(inputs.uniforms(4, 3, 1)).cuda()
    pos = torch.empty((4, 3), dtype=torch.int32, device="cuda")
    # M = 0 is a no-op
    assert L.ffs_sample(Ud.data_ptr(), 10, 3, 0, 0, None, None, None, None, 0, None) == 0
    # invalid shapes / dtype / workspace
    assert L.ffs_sample(Ud.data_ptr(), 10, 11, 0, 4, ud.data_ptr(), pos.data_ptr(), None, None, 0, None) == -1
    assert L.ffs_sample_marginal(Ud.data_ptr(), 10, 3, 0, 4, 4, ud.data_ptr(), pos.data_ptr(), None, None, 0, None) == -1
    assert L.ffs_sample(Ud.data_ptr(), 10, 3, 9, 4, ud.data_ptr(), pos.data_ptr(), None, None, 0, None) == -1
    # no / too small workspace: FFS_ENOWS
    assert L.ffs_sample(Ud.data_ptr(), 10, 3, 0, 4, ud.data_ptr(), pos.data_ptr(), None, None, 0, None) == ffs.FFS_ENOWS
    assert L.ffs_sample(None, 10, 3, 0, 4, ud.data_ptr(), pos.data_ptr(), None, None, 0, None) == -1
    # L beyond the supported range (16384 real, 8192 complex): FFS_EINVAL, never truncated
    # (calls with small N' go up to L = 2^18 on the tile-Gram path: test_tile_gram_path[_complex])
    assert L.ffs_workspace_bytes(16385, 256, 200, 0, 4) == 0
    assert L.ffs_workspace_bytes(16385, 8, 8, 0, 4) > 0
    assert L.ffs_workspace_bytes(262145, 8, 8, 0, 4) == 0
    assert L.ffs_workspace_bytes(8193, 256, 200, 1, 4) == 0
    assert L.ffs_workspace_bytes(8193, 8, 8, 1, 4) > 0
    assert L.ffs_workspace_bytes(262145, 8, 8, 1, 4) == 0
    assert L.ffs_sample(Ud.data_ptr(), 16385, 200, 0, 4, ud.data_ptr(), pos.data_ptr(), None, None, 0, None) == -1
    assert "unsupported L" in L.ffs_last_error().decode()
    # trace range outside [0, M)
    assert L.ffs_debug_trace(Ud.data_ptr(), 10, 3, 0, 4, 3, ud.data_ptr(), pos.data_ptr(), None, None, 0, None,
                             3, 2, pos.data_ptr()) == -1
    # caller-supplied outputs are validated by the binding
    with pytest.raises(ffs.FFSError):
        ffs.ffs_sample(Ud, ud, positions=torch.empty((4, 2), dtype=torch.int32, device="cuda"))
    with pytest.raises(ffs.FFSError):
        ffs.ffs_sample(Ud, ud, positions=torch.empty((4, 3), dtype=torch.int64, device="cuda"))
    # N = 1, N' = 1, L = N (full filling)
    for (l, n, np_) in [(9, 1, 1), (12, 5, 1), (6, 6, 6), (33, 33, 33)]:
        Ue = inputs.random_orthonormal(l, n, l + n)
        uni = inputs.uniforms(64, np_, 3)
        gpos, _, _ = run_gpu(Ue, uni, np_)
        rpos = ref.sample(Ue, uni, Np=np_)
        assert not compare_positions(Ue, uni, gpos, rpos, np_)["failures"]
        if l == n:
            assert all(sorted(p) == list(range(l)) for p in gpos.tolist())


@pytest.mark.parametrize("shape", ["dw", (40000, 24, 8, False), (20000, 16, 8, True)])
def test_host_path_matches_device_path(shape):
    ffs = _ffs()
    if shape == "dw":
        cfg = inputs.CONFIGS["dw"]
        U, Np = inputs.build_u(cfg), cfg.N
    else:  # beyond the panel kernels' L: the tile-Gram path through the host call
        L, N, Np, cx = shape
        U = inputs.random_orthonormal(L, N, L + N, complex_=cx)
    M = 20000  # > one host chunk
    uni = inputs.uniforms(M, Np, 77)
    dev, _, _ = run_gpu(U, uni, Np)
    hU = torch.from_numpy(U).pin_memory()
    hu = torch.from_numpy(uni).pin_memory()
    hp = ffs.ffs_sample_host(hU, hu, Np)
    assert (hp.numpy() == dev).all()


def test_library_is_the_native_one():
    import os
    ffs = _ffs()
    L = ffs.load()
    assert os.path.dirname(ffs.lib_path()).endswith("paper_2109_07358_b200")
    U = inputs.random_orthonormal(256, 32, 3)
    run_gpu(U, inputs.uniforms(16, 32, 3), 32)
    assert L.ffs_last_launch_count() >= 1


EXTREME = [(16, 4, 4, False), (256, 32, 32, False), (300, 33, 33, False), (1500, 19, 19, False),
           (5000, 11, 11, False), (2000, 9, 9, True), (64, 21, 9, True)]


@pytest.mark.parametrize("L,N,Np,cplx", EXTREME)
@pytest.mark.parametrize("useL", [0.0, 1.0 - 2.0 ** -53])
def test_extreme_selection_uniforms(L, N, Np, cplx, useL):
    """Selection uniforms at the ends of [0, 1): u = 0 selects the first site with w > 0 and
    u = 1 - 2^-53 the last one (reading Q5: strict C(x) > u*T, else the last positive-weight
    site). Both rules are deterministic, so positions must agree exactly (no tie exclusion);
    u -> 1 drives the kernels' no-crossing fallback paths."""
    U = inputs.random_orthonormal(L, N, 4242 + L + N, complex_=cplx)
    M = 40
    uni = inputs.uniforms(M, Np, 99 + L)
    uni[:, Np:] = useL
    gpos, gfl, _ = run_gpu(U, uni, Np)
    rpos = ref.sample(U, uni, Np=Np)
    assert (gpos == rpos).all(), np.argwhere(gpos != rpos)[:5]
    assert not (gfl & 1).any()


# Lockstep-dense path schedules (ffs_abi.cu launch_dense): several batches with a ragged last one,
# all-GEMM (theta 0) with each GEMM (Ozaki 8 slices as CTA pairs = default, Ozaki 8 slices one CTA
# per tile, Ozaki 7, DMMA), all-gathered (theta 1), the default hybrid, with and without the
# CUDA-graph driver; real and complex.
@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("opts", [{"dense_batch": 16}, {"dense_theta": 0}, {"dense_theta": 1},
                                  {"dense_batch": 7, "dense_theta": 0.5},
                                  {"dense_theta": 0, "dense_gemm": 7},
                                  {"dense_theta": 0, "dense_gemm": 0},
                                  {"dense_theta": 0.3, "graph": 0},
                                  {"dense_theta": 0, "gemm_2sm": 0},
                                  {"dense_theta": 0, "gemm_2sm": 3},
                                  {"dense_theta": 0.2, "gemm_2sm": 3, "dense_batch": 13},
                                  {"dense_theta": 0, "gram_draw": 0},
                                  {"dense_batch": 9, "dense_theta": 0.25, "gram_draw": 0},
                                  {"dense_theta": 0, "gram_kappa": 0},
                                  {"dense_theta": 0, "gj_pair": 0},
                                  {"dense_theta": 0.1, "gj_pair": 2},
                                  {"dense_theta": 0.6, "gram_draw": 3},
                                  {"dense_theta": 1, "gram_draw": 3, "dense_batch": 9},
                                  {"dense_theta": 0.4, "dense_batch": 5, "gj_pair": 0},
                                  {"dense_theta": 0, "gram_kappa": 1e30}])
def test_dense_path_schedules(opts, cplx):
    ffs = _ffs()
    for k, v in opts.items():
        ffs.set_option(k, v)
    L, N = 2100, 258  # L: 2 clusters' rows with a ragged tail; N' = N: ragged last panel block
    U = inputs.random_orthonormal(L, N, 77 + int(cplx), complex_=cplx)
    M = 40
    uni = inputs.uniforms(M, N, 4242)
    gpos, gflags, gw = run_gpu(U, uni, N, trace_S=2, trace_S0=M - 2)
    rpos = ref.sample(U, uni, Np=N)
    r = compare_positions(U, uni, gpos, rpos, N)
    assert not r["failures"], r["failures"][:3]
    assert (gflags == 0).all()
    _, rw = ref.weights(U, uni[M - 2:], Np=N)
    assert compare_weights(gw, rw, gpos[M - 2:], rpos[M - 2:]) <= WEIGHT_TOL


# Gram draws (ffs_gram.cuh) at the ends of [0, 1): u = 0 takes the first site with w > 0, u = 1 - 2^-53
# the last one -- exactly, through the tile totals (Gram forms or direct sums) and the in-tile scan.
@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("kappa", [1e3, 0.0])
@pytest.mark.parametrize("useL", [0.0, 1.0 - 2.0 ** -53])
def test_gram_draw_extreme_uniforms(useL, kappa, cplx):
    ffs = _ffs()
    ffs.set_option("dense_theta", 0)
    ffs.set_option("gram_kappa", kappa)
    L, N = 2100, 258
    U = inputs.random_orthonormal(L, N, 911 + int(cplx), complex_=cplx)
    M = 12
    uni = inputs.uniforms(M, N, 31)
    uni[:, N:] = useL
    ffs.ffs_gram_counters(reset=True)
    gpos, gfl, _ = run_gpu(U, uni, N)
    draws, direct = ffs.ffs_gram_counters()
    assert draws == M * N
    # kappa = 0 sends every draw through the direct tile totals; at these extreme uniforms the
    # pivots are the first / last sites with any weight (often tiny: large |d|), so the guard also
    # fires often with the default kappa
    assert direct >= draws if kappa == 0.0 else direct <= draws
    rpos = ref.sample(U, uni, Np=N)
    assert (gpos == rpos).all(), np.argwhere(gpos != rpos)[:5]
    assert not (gfl & 1).any()


def test_graph_replay_matches_direct_launches():
    """The CUDA-graph driver replays the captured block loop: a second call with the same buffers
    (graph reuse) and a call with new buffers (graph update) give the direct-launch result."""
    ffs = _ffs()
    L, N, M = 2100, 258, 24
    U = _to_dev(inputs.random_orthonormal(L, N, 5))
    outs = []
    for graph in (0, 1, 1):
        ffs.set_option("graph", graph)
        ud = torch.from_numpy(inputs.uniforms(M, N, 11)).cuda()
        outs.append(ffs.ffs_sample(U, ud).cpu().numpy())
    assert (outs[0] == outs[1]).all() and (outs[1] == outs[2]).all()
    assert ffs.ffs_last_launch_count() > 10  # kernel nodes of the replayed graph


def test_options_api():
    ffs = _ffs()
    assert ffs.get_option("dense_gemm") == 8.0
    ffs.set_option("dense_gemm", 7)
    assert ffs.get_option("dense_gemm") == 7.0
    ffs.set_option("dense_gemm", float("nan"))
    assert ffs.get_option("dense_gemm") == 8.0
    lib = ffs.load()
    assert lib.ffs_set_option(99, 1.0) == ffs.FFS_EINVAL
    ffs.set_option("dense_gemm", 5)  # accepted here, rejected when a plan is made
    U = _to_dev(inputs.random_orthonormal(2100, 258, 5))
    with pytest.raises(ffs.FFSError):
        ffs.ffs_sample(U, torch.from_numpy(inputs.uniforms(4, 258, 1)).cuda())


# Marginals at large L run the step + batched-GJ kernels with every block contracted gathered
# (ffs_abi.cu dense_eligible); option large_l_marginal = 0 keeps them on the per-sample cluster kernel.
@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("step", ["1", "0"])
def test_large_L_marginal_paths(step, cplx):
    _ffs().set_option("large_l_marginal", int(step))
    L, N, Np = 2100, 300, 42  # ragged last block (42 = 5 x 8 + 2)
    U = inputs.random_orthonormal(L, N, 91 + int(cplx), complex_=cplx)
    uni = inputs.uniforms(64, Np, 515)
    gpos, gflags, gw = run_gpu(U, uni, Np, trace_S=2)
    rpos = ref.sample(U, uni, Np=Np)
    r = compare_positions(U, uni, gpos, rpos, Np)
    assert not r["failures"], r["failures"][:3]
    assert (gflags == 0).all()
    _, rw = ref.weights(U, uni[:2], Np=Np)
    assert compare_weights(gw, rw, gpos, rpos) <= WEIGHT_TOL


# Degenerate marginals (N' = 1: one draw with w(x) = |U[x, m_1]|^2; N' = 2: one GJ-free block)
# on every path: warp (L <= 256), CTA owner, cluster (N < 256), block-step (N >= 256).
@pytest.mark.parametrize("L,N,Np,cplx", [
    (200, 30, 1, False), (300, 40, 1, False), (300, 40, 2, True), (2100, 9, 1, False), (2100, 9, 2, True),
    (2100, 300, 1, False), (2100, 300, 2, True), (4096, 256, 9, False),
])
def test_degenerate_marginals(L, N, Np, cplx):
    U = inputs.random_orthonormal(L, N, 7 * L + N, complex_=cplx)
    uni = inputs.uniforms(48, Np, L + 3 * N)
    gpos, gflags, gw = run_gpu(U, uni, Np, trace_S=2)
    rpos = ref.sample(U, uni, Np=Np)
    r = compare_positions(U, uni, gpos, rpos, Np)
    assert not r["failures"], r["failures"][:3]
    assert (gflags == 0).all()
    _, rw = ref.weights(U, uni[:2], Np=Np)
    assert compare_weights(gw, rw, gpos, rpos) <= WEIGHT_TOL
    if Np == 1:  # the first conditional is |U[x, m_1]|^2 exactly (Eq. 3 with k = 1)
        m1 = np.floor(uni[:2, 0] * N).astype(int)
        for s in range(2):
            ref_w = np.abs(U[:, m1[s]]) ** 2
            assert np.max(np.abs(gw[s, 0] - ref_w / ref_w.sum())) <= 1e-13


# Large-L full sampling with very few samples (a batch far below the GEMM's 128-column tile) and
# with an odd N (not dense-eligible: the per-sample cluster kernel).
@pytest.mark.parametrize("L,N,M,cplx", [(2100, 256, 1, False), (2100, 256, 3, True), (2100, 257, 5, False)])
def test_large_L_small_batches(L, N, M, cplx):
    U = inputs.random_orthonormal(L, N, 3 * L + N + M, complex_=cplx)
    uni = inputs.uniforms(M, N, 99 + M)
    gpos, gflags, gw = run_gpu(U, uni, N, trace_S=1)
    rpos = ref.sample(U, uni, Np=N)
    r = compare_positions(U, uni, gpos, rpos, N)
    assert not r["failures"], r["failures"][:3]
    assert (gflags == 0).all()
    _, rw = ref.weights(U, uni[:1], Np=N)
    assert compare_weights(gw, rw, gpos, rpos) <= WEIGHT_TOL


# Odd N' on the block-step marginal path (the batched Gauss-Jordan kernel's W rows are then not
# 16-byte aligned: element-wise accesses), several block counts and a ragged last block.
@pytest.mark.parametrize("Np", [19, 21, 43])
def test_block_step_odd_marginal(Np):
    L, N = 2100, 300
    U = inputs.random_orthonormal(L, N, 3 * Np)
    M = 48
    uni = inputs.uniforms(M, Np, 17 + Np)
    gpos, gflags, gw = run_gpu(U, uni, Np, trace_S=2, trace_S0=M - 2)
    rpos = ref.sample(U, uni, Np=Np)
    r = compare_positions(U, uni, gpos, rpos, Np)
    assert not r["failures"], r["failures"][:3]
    assert (gflags == 0).all()
    _, rw = ref.weights(U, uni[M - 2:], Np=Np)
    assert compare_weights(gw, rw, gpos[M - 2:], rpos[M - 2:]) <= WEIGHT_TOL


# The tile-Gram path (ffs_kmarg.cuh) takes every real shape with N' <= 64 and 64 N' <= 3 L by
# default; with the option off the same shapes run on the panel kernels (CTA owner, cluster,
# block-step), which stay covered here -- including the extreme selection uniforms.
PANEL_SHAPES = [(1024, 40, 21), (1500, 19, 19), (5000, 11, 11), (9000, 7, 7), (2100, 300, 42), (2100, 300, 19),
                (2100, 300, 1), (4096, 256, 9)]


@pytest.mark.parametrize("L,N,Np", PANEL_SHAPES)
def test_panel_paths_without_tile_gram(L, N, Np):
    _ffs().set_option("tile_gram", 0)
    U = inputs.random_orthonormal(L, N, 31 * L + N)
    M = 48
    uni = inputs.uniforms(M, Np, L + N + Np)
    gpos, gflags, gw = run_gpu(U, uni, Np, trace_S=2, trace_S0=M - 2)
    rpos = ref.sample(U, uni, Np=Np)
    r = compare_positions(U, uni, gpos, rpos, Np)
    assert not r["failures"], r["failures"][:3]
    assert (gflags == 0).all()
    _, rw = ref.weights(U, uni[M - 2:], Np=Np)
    assert compare_weights(gw, rw, gpos[M - 2:], rpos[M - 2:]) <= WEIGHT_TOL
    for useL in (0.0, 1.0 - 2.0 ** -53):
        uni[:, Np:] = useL
        gpos, gfl, _ = run_gpu(U, uni, Np)
        assert (gpos == ref.sample(U, uni, Np=Np)).all()
        assert not (gfl & 1).any()


# Tile-Gram path: tile sizes of 1, 3, 4 and 16 rows per lane (L = 1024 .. 16384, ragged last tiles),
# N' from 1 to 64, full sampling (N' = N) and marginals, many samples per warp slot.
@pytest.mark.parametrize("L,N,Np", [(600, 20, 20), (1024, 128, 16), (2500, 64, 48), (3000, 300, 57), (4096, 140, 64),
                                   (16384, 96, 33), (7000, 12, 1), (8192, 200, 96), (200, 60, 5), (256, 90, 8),
                                   (40000, 24, 8), (70001, 16, 5)])
@pytest.mark.parametrize("mode", [1, 2, 3, 4])  # default (flat forms for N' <= 24, else blocked; half-warp owners for L <= 1024), flat, blocked, warp owners
def test_tile_gram_path(L, N, Np, mode):
    ffs = _ffs()
    if mode == 2 and Np > 64:
        pytest.skip("flat forms keep N'(N'+1)/2 offsets and coefficients per owner in shared memory: N' <= 64")
    ffs.set_option("tile_gram", mode)
    assert ffs.ffs_workspace_bytes(L, N, Np, ffs.FFS_F64, 1) > 16 * N * N * 8  # the tile-Gram plan (holds K)
    U = inputs.random_orthonormal(L, N, 13 * L + N)
    M = 3000 if L * Np <= 40000 else 96
    uni = inputs.uniforms(M, Np, 5 * L + Np)
    gpos, gflags, gw = run_gpu(U, uni, Np, trace_S=2, trace_S0=M - 2)
    n_ref = min(M, 96)
    idx = np.array(_spread(M, n_ref))
    rpos = ref.sample(U, uni[idx], Np=Np)
    r = compare_positions(U, uni[idx], gpos[idx], rpos, Np)
    assert not r["failures"], r["failures"][:3]
    assert (gflags == 0).all()
    assert all(len(set(q)) == Np for q in gpos.tolist())
    last = np.arange(M - 2, M)
    rlast, rw = ref.weights(U, uni[last], Np=Np)
    assert compare_weights(gw, rw, gpos[last], rlast) <= WEIGHT_TOL
    for useL in (0.0, 1.0 - 2.0 ** -53):
        uni2 = uni[:32].copy()
        uni2[:, Np:] = useL
        gpos2, gfl2, _ = run_gpu(U, uni2, Np)
        assert (gpos2 == ref.sample(U, uni2, Np=Np)).all()
        assert not (gfl2 & 1).any()


# Complex tile-Gram path (ffs_kmarg_c.cuh: Hermitian tile Gram matrices, flat forms, N' <= 32): half-warp
# and warp owners, 1 / 3 / 4 / 6 rows per lane and the chunked row scan beyond L = 16384, marginals and full sampling, extreme selection uniforms;
# and the same shapes on the panel kernels with the option off.
@pytest.mark.parametrize("L,N,Np", [(600, 20, 20), (1024, 64, 16), (2500, 40, 32), (4096, 300, 24), (3000, 12, 1),
                                    (6000, 16, 8), (20000, 16, 8), (40001, 12, 5)])
@pytest.mark.parametrize("mode", [1, 0])
def test_tile_gram_path_complex(L, N, Np, mode):
    ffs = _ffs()
    if mode == 0 and L > 8192:
        pytest.skip("the complex panel kernels stop at L = 8192")
    ffs.set_option("tile_gram", mode)
    U = inputs.random_orthonormal(L, N, 17 * L + N, complex_=True)
    M = 2000 if (mode == 1 and L * Np <= 40000) else 64
    uni = inputs.uniforms(M, Np, 3 * L + Np)
    gpos, gflags, gw = run_gpu(U, uni, Np, trace_S=2, trace_S0=M - 2)
    idx = np.array(_spread(M, min(M, 64)))
    rpos = ref.sample(U, uni[idx], Np=Np)
    r = compare_positions(U, uni[idx], gpos[idx], rpos, Np)
    assert not r["failures"], r["failures"][:3]
    assert (gflags == 0).all()
    assert all(len(set(q)) == Np for q in gpos.tolist())
    last = np.arange(M - 2, M)
    rlast, rw = ref.weights(U, uni[last], Np=Np)
    assert compare_weights(gw, rw, gpos[last], rlast) <= WEIGHT_TOL
    for useL in (0.0, 1.0 - 2.0 ** -53):
        uni2 = uni[:32].copy()
        uni2[:, Np:] = useL
        gpos2, gfl2, _ = run_gpu(U, uni2, Np)
        assert (gpos2 == ref.sample(U, uni2, Np=Np)).all()
        assert not (gfl2 & 1).any()
