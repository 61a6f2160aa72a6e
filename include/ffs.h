/* ffs.h — C ABI of the B200-native fast fermion sampling (FFS) hot path (libffs.so).
 *
 * The operation (arXiv 2109.07358, PAPER.md):
 *   Given U (L x N, orthonormal columns, U^dagger U = 1), draw ordered
 *   configurations x = (x_1..x_N) from P(x) = |det U_{x,n}|^2 / N!  (Eq. 1)
 *   by the FFS algorithm: a uniformly random permutation m of the columns, then
 *   for k = 1..N the conditional P(x_k | x_1..x_{k-1}; m) ∝ |u_{x_k}^T h|^2, h the normal vector
 *   of u_{x_1..x_{k-1}} in the span of columns m_1..m_k (Eq. 3), drawn by inverse
 *   CDF. The marginal variant stops after N' < N steps.
 *
 * Conventions shared with the oracle (readings Q3-Q8):
 *   - dtype FFS_F64: U is double[L][N] row-major. FFS_C128: U is interleaved (re,im) double[L][N][2];
 *     u_x^T h is BILINEAR (no conjugation), weights are |.|^2.
 *   - uniforms: double[M][2N'] in [0,1). Row i: [0, N') drive the permutation draw (forward partial
 *     Fisher-Yates: m = (0..N-1); for j < N': n = N-j, r = j + min(n-1, floor(u[j]*n)),
 *     swap(m[j], m[r])); [N', 2N') are the N' selection uniforms.
 *   - selection at step k with weights w >= 0 (chosen sites forced to 0): T = sum of w;
 *     x_k = min{x : C(x) > u*T, w(x) > 0}, C the inclusive prefix sum in index order;
 *     if none, the largest x with w(x) > 0.
 *   - positions: int32[M][N'] out, 0-based site indices, in sampling order.
 *   - sample_flags (optional, may be NULL): int32[M] out; bit0 = some step had a non-finite or
 *     non-positive total T; bit1 = a selected normalised weight was < 1e-12. Numerical conditions
 *     never abort a call.
 *
 * Ownership / memory: every pointer of the device entry points is a DEVICE pointer owned by the
 * caller; the library allocates nothing (the caller provides `workspace` of at least
 * ffs_workspace_bytes(...) bytes, 256-byte aligned). Calls are asynchronous on `stream` and
 * re-entrant across streams with distinct workspaces. U orthonormality is the caller's
 * precondition and is not checked.
 *
 * Errors (all synchronous, message in ffs_last_error()): FFS_EINVAL for null pointers when M > 0,
 * N < 1, N > L, N' not in [1, N], unknown dtype, or L beyond the supported range (L <= 16384 real,
 * L <= 8192 complex: one sample's L x 8 panel must fit the register files of one thread-block
 * cluster / one SM; calls with small N' -- the tile-Gram path, FFS_OPT_TILE_GRAM -- keep no
 * panel and go up to L = 262144; any other larger L returns FFS_EINVAL, it is never truncated); FFS_ENOWS if the workspace
 * is NULL or smaller than ffs_workspace_bytes(...); FFS_ECUDA for CUDA launch/runtime errors.
 * M == 0 is an OK no-op.
 */
#ifndef FFS_H
#define FFS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { FFS_F64 = 0, FFS_C128 = 1 } ffs_dtype;
typedef enum { FFS_OK = 0, FFS_EINVAL = -1, FFS_ECUDA = -2, FFS_ENOWS = -3 } ffs_status;

/* Device workspace bytes needed by ffs_sample / ffs_sample_marginal / ffs_debug_trace on the
 * current CUDA device. Returns 0 for invalid arguments. Size depends on the path the call takes:
 * small for L <= 256 (permutations only); for L >= 2048 with N >= 256 (the lockstep block-step
 * path) it holds, per batch of S samples (the most whose factors W [N'][N'] fit a
 * 24 GB budget, at least 1024 and at most 8192, at most M), every batch sample's W, the coefficient
 * and panel matrices Y [N][8 S] and P [L][8 S] of the dense GEMM, U^T and the permutations: e.g.
 * 9.4 GB for the C5 config (L=16384, N=1024, M=1024), 20 GB for C4 (L=4096, N=512, c128). On the
 * tile-Gram path (real U, small N'; FFS_OPT_TILE_GRAM) it holds U^T, the tile Gram matrices of U
 * (8 G N^2 bytes, G = 16 or 32 tiles), the permutations and, for N' > 32, one N' x N' coefficient
 * matrix per resident sample owner: 0.4 GB for the C5 marginal (N' = 64). */
size_t ffs_workspace_bytes(int64_t L, int64_t N, int64_t Nprime, ffs_dtype dtype, int64_t M);

/* Full sampling (N' = N): Eq. 1-3. uniforms [M][2N], positions [M][N]. */
int ffs_sample(const void* U, int64_t L, int64_t N, ffs_dtype dtype, int64_t M,
               const double* uniforms, int32_t* positions, int32_t* sample_flags,
               void* workspace, size_t ws_bytes, void* stream);

/* Marginal sampling of N' <= N particles: the same chain stopped after N' steps.
 * uniforms [M][2N'], positions [M][N']. */
int ffs_sample_marginal(const void* U, int64_t L, int64_t N, ffs_dtype dtype, int64_t M, int64_t Nprime,
                        const double* uniforms, int32_t* positions, int32_t* sample_flags,
                        void* workspace, size_t ws_bytes, void* stream);

/* As ffs_sample_marginal, and also writes the normalised conditional weight vectors (Eq. 3,
 * w(x)/T per step) of samples S0 .. S0+S-1 along their own path: weights double[S][N'][L]
 * (DEVICE). The traced samples run in the same launch configuration as every other sample, so a
 * trace of the last samples checks the last tiles/clusters/batches. FFS_EINVAL if S0 < 0, S < 0 or
 * S0 + S > M. */
int ffs_debug_trace(const void* U, int64_t L, int64_t N, ffs_dtype dtype, int64_t M, int64_t Nprime,
                    const double* uniforms, int32_t* positions, int32_t* sample_flags,
                    void* workspace, size_t ws_bytes, void* stream, int64_t S0, int64_t S, double* weights);

/* Host-buffer entry point (end-to-end path): U, uniforms, positions, sample_flags are HOST
 * pointers (pinned memory recommended); the call copies inputs host->device, samples, copies the
 * results device->host and returns after the results are in host memory. `workspace` is a DEVICE
 * buffer of at least ffs_host_workspace_bytes(...) bytes. Samples are processed in chunks so that
 * the copies of one chunk overlap the sampling of another. */
size_t ffs_host_workspace_bytes(int64_t L, int64_t N, int64_t Nprime, ffs_dtype dtype, int64_t M);
int ffs_sample_host(const void* U, int64_t L, int64_t N, ffs_dtype dtype, int64_t M, int64_t Nprime,
                    const double* uniforms, int32_t* positions, int32_t* sample_flags,
                    void* workspace, size_t ws_bytes, void* stream);

/* L-ensemble DPP front end (text-summarisation pipeline step 2). The caller has
 * eigendecomposed the correlation matrix C = sum_j lambda_j v_j v_j^dagger (setup, not part of the
 * path). Per sample i, eigenvector j is kept iff keep_u[j] < lambda_j/(lambda_j + 1) (the paper's
 * "selected with probability lambda_j/(lambda_j+1)"; the decision is taken in fp64); the kept
 * columns, in ascending j, form U_i (L x N_i), which is sampled by FFS exactly as ffs_sample
 * samples U (Eq. 1-3) with N = N_i. The sampled subsets follow the L-ensemble law
 * P(S) = det(C_S) / det(I + C).
 *   V        : DEVICE [L][K] eigenvectors (orthonormal columns), dtype as ffs_sample; K <= L
 *   lambda   : DEVICE double[K], eigenvalues >= 0
 *   uniforms : DEVICE double[M][3K]: [0,K) keep draws, [K,2K) the permutation draws of U_i
 *              (first N_i used, rule of ffs_sample with N = N_i), [2K,3K) the N_i selections
 *   positions: DEVICE int32[M][K] out, sampling order; entries k >= N_i are -1
 *   counts   : DEVICE int32[M] out (N_i) or NULL; sample_flags as ffs_sample (NULL allowed)
 * Workspace: ffs_lensemble_workspace_bytes(L, K, dtype, M) bytes (0 = invalid arguments).
 * Errors as ffs_sample (L <= 16384 real / 8192 complex). An empty kept set gives N_i = 0. */
size_t ffs_lensemble_workspace_bytes(int64_t L, int64_t K, ffs_dtype dtype, int64_t M);
int ffs_sample_lensemble(const void* V, const double* lambda, int64_t L, int64_t K, ffs_dtype dtype, int64_t M,
                         const double* uniforms, int32_t* positions, int32_t* counts, int32_t* sample_flags,
                         void* workspace, size_t ws_bytes, void* stream);

/* Continuous / large-L variant (Supp S7): the permutation, elimination and
 * normal vector of ffs_sample, but x_k is drawn by a Metropolis chain of Mcond updates instead of
 * the inverse-CDF draw over all L sites ("accepted with probability |u_{x_k+dx}^T h|^2 /
 * |u_{x_k}^T h|^2", "iterated for M_cond times"; for large L "a discrete update x_k -> x_k'"), so
 * the cost per sample is O(N'^3 + Mcond N'^2), independent of L. Readings shared with the oracle
 * (Q16-Q18): the chain of step k starts at x = floor(u_init L); each update proposes
 * x' = floor(u_prop L) (uniform, symmetric) and accepts iff u_acc w(x) < w(x'); chosen sites have
 * w = 0. The result approaches Eq. 1 as Mcond grows (exact only in that limit).
 *   uniforms : DEVICE double[M][N' + N'(1 + 2 Mcond)]: [0, N') permutation draws (rule of
 *              ffs_sample), then per step k: u_init, (u_prop, u_acc) x Mcond
 *   positions: DEVICE int32[M][N'] out; sample_flags (or NULL): bit0 = non-finite pivot,
 *              bit2 = a chain ended on a zero-weight site (Mcond too small)
 * Any L <= 2^31-1 (U is only read at the proposed rows); N' <= N <= L; Mcond <= 4096.
 * Workspace: ffs_metropolis_workspace_bytes(...) bytes. Errors as ffs_sample. */
size_t ffs_metropolis_workspace_bytes(int64_t L, int64_t N, int64_t Nprime, int64_t Mcond, ffs_dtype dtype, int64_t M);
int ffs_sample_metropolis(const void* U, int64_t L, int64_t N, ffs_dtype dtype, int64_t M, int64_t Nprime,
                          int64_t Mcond, const double* uniforms, int32_t* positions, int32_t* sample_flags,
                          void* workspace, size_t ws_bytes, void* stream);

/* Modified-HKPV sampler, the paper's comparison method ("O(N^2 L) with certain
 * modification", :81 "the modified HPKV algorithm requires 2LN^2 operations"; its steps as
 * SPEC.md:238-246): the chain rule on K = U U^dagger. Residuals r(x) = |u_x|^2 - sum_j |<u_x, e_j>|^2;
 * step k draws x_k ∝ r (selection rule of ffs_sample: strict C(x) > u T, chosen sites and
 * non-positive residuals weigh 0), orthonormalises u_{x_k} against the earlier e_j (Gram-Schmidt,
 * Hermitian inner product) and subtracts |<u_x, e_k>|^2 from every residual. It samples the same
 * law as ffs_sample (Eq. 1) with different conditionals and no permutation; provided to measure
 * the paper's "about 100% more efficient" claim on the same GPU (bench.py extensions).
 *   uniforms : DEVICE double[M][N'] selection draws; positions DEVICE int32[M][N'] out (sampling
 *              order); sample_flags as ffs_sample (NULL allowed)
 * Same shapes and errors as ffs_sample_marginal; workspace ffs_hkpv_workspace_bytes(...) bytes. */
size_t ffs_hkpv_workspace_bytes(int64_t L, int64_t N, int64_t Nprime, ffs_dtype dtype, int64_t M);
int ffs_sample_hkpv(const void* U, int64_t L, int64_t N, ffs_dtype dtype, int64_t M, int64_t Nprime,
                    const double* uniforms, int32_t* positions, int32_t* sample_flags, void* workspace,
                    size_t ws_bytes, void* stream);

/* Observables of FFS samples, on the device (Supp S5).
 * positions: DEVICE int32[M][N'] as written by the sampling calls; entries < 0 (the L-ensemble's
 * padding) are skipped. Outputs are DEVICE arrays, zeroed and filled by the call (async on stream).
 *   ffs_occupation      : occ[x] = number of samples with site x occupied, x < L (uint64[L]);
 *                         <n_x> = occ[x] / M ("occupation number").
 *   ffs_pair_occupation : pair[x][y] = number of samples with x and y both occupied, x, y < W
 *                         (uint64[W][W]; the diagonal is occ); <n_x n_y> = pair / M.
 *   ffs_gutzwiller_reweight: Slater-Jastrow reweighting with the Gutzwiller factor of Eq. 4,
 *                         J = exp(-V/2 sum_i n_{i,up} n_{i,down}): a spinful sample s is the pair of
 *                         rows (2s, 2s+1) = (up, down), D_s = number of sites in both rows,
 *                         J_s^2 = exp(-V D_s); result (DOUBLE[2 + L]): [0] = <J^2>_0 =
 *                         (1/Ms) sum_s J_s^2, [1] = <D>_J, [2 + x] = <n_x>_J (both spins), with
 *                         <O>_J = sum_s J_s^2 O_s / sum_s J_s^2 (the paper's <J^2 o_L>_0/<J^2>_0).
 *                         dcount (uint64[N'+1], or NULL) receives the histogram of D_s. The sums
 *                         are formed from exact integer histograms by D (order-independent).
 *                         Ms >= 1 spinful samples (2 Ms rows); workspace of
 *                         ffs_gutzwiller_workspace_bytes(N', L) bytes (FFS_ENOWS if smaller).
 * Errors: FFS_EINVAL for null pointers / invalid sizes (W <= 46340, N' <= 8192 for pairs), FFS_ECUDA. */
int ffs_occupation(const int32_t* positions, int64_t M, int64_t Nprime, int64_t L, unsigned long long* occ,
                   void* stream);
int ffs_pair_occupation(const int32_t* positions, int64_t M, int64_t Nprime, int64_t W, unsigned long long* pair,
                        void* stream);
size_t ffs_gutzwiller_workspace_bytes(int64_t Nprime, int64_t L);
int ffs_gutzwiller_reweight(const int32_t* positions, int64_t Ms, int64_t Nprime, int64_t L, double V, double* result,
                            unsigned long long* dcount, void* workspace, size_t ws_bytes, void* stream);

/* Number of kernel launches the last successful sampling call on this thread issued. */
int ffs_last_launch_count(void);

/* Measurement hooks (bench.py): when enabled, each device sampling call records CUDA events on
 * its stream immediately before and after its dominant kernel (the per-sample sampling kernel);
 * ffs_last_kernel_ms() waits for the last call's end event and returns the elapsed milliseconds
 * (-1 if none). Per calling thread. */
int ffs_profile_enable(int on);
float ffs_last_kernel_ms(void);

/* Tuning options (process-wide; read when a call plans its launch, so they apply to later calls).
 * Defaults are the measured best; tests use them to drive every schedule of a path.
 * ffs_set_option returns FFS_OK, or FFS_EINVAL for an unknown option; a NaN value restores the
 * default. ffs_get_option returns the current value (NaN for an unknown option). */
typedef enum {
  FFS_OPT_DENSE_GEMM = 1,       /* full sampling at large L, blocks with k0 >= theta N': the GEMM P = U Y
                                   8 = Ozaki FP64 emulation on the INT8 tensor cores, 8 slices (default;
                                       normwise panel error <= 1.3e-15, fp64 level)
                                   7 = the same with 7 slices (<= 2.2e-13)
                                   0 = FP64 DMMA (mma.sync m8n8k4) */
  FFS_OPT_DENSE_THETA = 2,      /* gathered/GEMM crossover fraction theta; < 0 = default */
  FFS_OPT_DENSE_BATCH = 3,      /* samples per lockstep batch of the block-step paths; 0 = default */
  FFS_OPT_BLOCK_STEP = 4,       /* 1 (default): L >= 2048, even N >= 256 on the block-step paths;
                                   0: the per-sample cluster kernel */
  FFS_OPT_LARGE_L_MARGINAL = 5, /* 1 (default): large-L marginals on the block-step kernels;
                                   0: the per-sample cluster kernel */
  FFS_OPT_CLUSTER = 6,          /* 1 (default): L >= 2048 on cluster kernels; 0: one CTA per sample */
  FFS_OPT_GRAPH = 7,            /* 1 (default): the block-step paths' launches are captured once and
                                   replayed as a CUDA graph (not while the caller's stream is being
                                   captured); 0: direct launches */
  FFS_OPT_FORCE_GENERIC = 8,    /* 1: every shape on the per-sample warp/CTA-owner kernel (testing) */
  FFS_OPT_GEMM_2SM = 9,         /* 1 (default): the 8-slice Ozaki GEMM runs as CTA pairs (tcgen05
                                   cta_group::2) on 256 x 128 tiles in two passes of four diagonals;
                                   3: CTA pairs on 256 x 64 tiles, one pass; 0: one CTA per 128 x 64 tile */
  FFS_OPT_GRAM_DRAW = 10,       /* 1 (default): the draws of a GEMM block step run one warp per sample on
                                   the tile Gram matrices of the panel (ffs_gram.cuh) -- also the
                                   gathered blocks, whose panel the cluster kernel then only contracts
                                   (3: gathered blocks draw in the cluster kernel);
                                   0: the cluster step kernel (panel in registers) */
  FFS_OPT_GRAM_KAPPA = 11,      /* Gram draws: recompute the tile totals directly from the panel when
                                   T < bound / kappa (cancellation guard); default 1e4 */
  FFS_OPT_DENSE_MIN_L = 12,     /* smallest L on the block-step paths (default 2048); below 2048 every
                                   block of a full sampling call takes the GEMM + Gram draws */
  FFS_OPT_DENSE_MIN_N = 13,     /* smallest N on the block-step paths (default 256) */
  FFS_OPT_TILE_GRAM = 14,       /* 1 (default): complex U with N' <= 32 (N <= 1024) and real U, L <= 262144, 64 N' <= 3 L and N' <= 24 (L <= 1024), 32 (L < 2048), 64 (L < 4096), 96 (larger L): the tile-Gram
                                   path (ffs_kmarg.cuh): tile totals as quadratic forms of the 32 tile
                                   Gram matrices of U, one warp per sample; 0: the panel kernels */
  FFS_OPT_GJ_PAIR = 15,         /* 1 (default): real block-step paths update W for two consecutive blocks in
                                   one pass (ffs_dense_gj2_kernel: half the W traffic); 2: complex too;
                                   0: one pass per block */
  FFS_OPT_LAST = 15
} ffs_option;
int ffs_set_option(int option, double value);
double ffs_get_option(int option);

/* Diagnostics of the Gram draws (process-wide device counters, read synchronously): out[0] =
 * draws taken by ffs_gram_draw_kernel since the last reset, out[1] = draws whose tile totals were
 * recomputed directly from the panel (cancellation guard / degenerate totals). reset != 0 zeroes
 * the counters after reading. Returns FFS_OK or FFS_ECUDA. */
int ffs_gram_counters(unsigned long long out[2], int reset);

/* Thread-local message for the last non-OK return on this thread ("" if none). */
const char* ffs_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* FFS_H */
