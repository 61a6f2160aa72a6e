/* ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU implementation of the fast fermion sampling (FFS)
 * algorithm of arXiv 2109.07358 exactly as the paper states it: a random permutation m
 * (PAPER.md:69), then for k = 1..N the conditional P(x_k | x_1..x_{k-1}; m) ∝ |u_{x_k}^T h|^2
 * with h the unit normal vector of u_{x_1..x_{k-1}} (Eq. 3), h obtained by the
 * iterative Gaussian elimination of Supp S1, and an inverse-CDF draw.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
 * load this library. It shares no code, header, table or helper with the CUDA path
 * (paper_2109_07358_b200/csrc); the CUDA path never calls it.
 *
 * fp64 throughout; complex U as C99 double _Complex (interleaved re,im — identical bytes to the
 * ABI's C128 layout). OpenMP only across independent samples.
 *
 * Build: gcc -O2 -fopenmp -shared -fPIC -o libffs_ref.so ffs_ref.c -lm
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define FFS_REF_F64 0
#define FFS_REF_C128 1

/* ---- real instantiation ---- */
#define SCALAR double
#define ABS2(z) ((z) * (z))
#define CONJ(z) (z)
#define SFX(name) name##_f64
#include "ffs_ref_core.h"
#undef SCALAR
#undef ABS2
#undef CONJ
#undef SFX

/* ---- complex instantiation ---- */
static inline double abs2_c(double _Complex z) { return creal(z) * creal(z) + cimag(z) * cimag(z); }
#define SCALAR double _Complex
#define ABS2(z) abs2_c(z)
#define CONJ(z) conj(z)
#define SFX(name) name##_c128
#include "ffs_ref_core.h"
#undef SCALAR
#undef ABS2
#undef CONJ
#undef SFX

/* Permutation draw ("generate a vector m as a random permutation of n"; reading Q6):
 * forward partial Fisher-Yates over the first Np slots:
 *   m = (0..N-1); for j = 0..Np-1: n = N-j; r = j + min(n-1, floor(u[j]*n)); swap(m[j], m[r]). */
void ffs_ref_permutation(const double* u, int64_t N, int64_t Np, int32_t* m)
{
    for (int64_t j = 0; j < N; ++j) m[j] = (int32_t)j;
    for (int64_t j = 0; j < Np; ++j) {
        int64_t n = N - j;
        int64_t r = (int64_t)floor(u[j] * (double)n);
        if (r > n - 1) r = n - 1;
        r += j;
        int32_t t = m[j];
        m[j] = m[r];
        m[r] = t;
    }
}

static int check_args(const double* U, int64_t L, int64_t N, int dtype, int64_t Np)
{
    if (!U || L < 1 || N < 1 || N > L || Np < 1 || Np > N) return -1;
    if (dtype != FFS_REF_F64 && dtype != FFS_REF_C128) return -1;
    return 0;
}

static size_t scratch_bytes(int64_t L, int64_t N, int64_t Np, int dtype)
{
    size_t es = dtype == FFS_REF_C128 ? 16 : 8;
    return es * (size_t)(Np * Np + Np) + 8 * (size_t)L + (size_t)L + 4 * (size_t)N + 64;
}

static int run_one(const double* U, int64_t L, int64_t N, int dtype, int64_t Np, const double* urow,
                   const int32_t* forced_m, const int32_t* forced_x, int32_t* x_out, double* w_trace,
                   double* hn2, double* tot, char* buf)
{
    size_t es = dtype == FFS_REF_C128 ? 16 : 8;
    char* p = buf;
    void* R = p;            p += es * (size_t)(Np * Np);
    void* h = p;            p += es * (size_t)Np;
    double* w = (double*)p; p += 8 * (size_t)L;
    char* chosen = p;       p += (size_t)L;
    int32_t* m = (int32_t*)(((uintptr_t)p + 3) & ~(uintptr_t)3);
    if (forced_m) memcpy(m, forced_m, 4 * (size_t)N);
    else ffs_ref_permutation(urow, N, Np, m);
    const double* usel = urow ? urow + Np : NULL;
    if (dtype == FFS_REF_F64)
        return sample_chain_f64(U, L, N, Np, m, usel, forced_x, x_out, w_trace, hn2, tot,
                                (double*)R, (double*)h, w, chosen);
    return sample_chain_c128((const double _Complex*)U, L, N, Np, m, usel, forced_x, x_out, w_trace,
                             hn2, tot, (double _Complex*)R, (double _Complex*)h, w, chosen);
}

/* ffs_ref_sample_marginal: M independent samples of Np steps (Np = N: full sampling).
 * uniforms [M][2Np] (perm draws | selection draws), positions [M][Np], flags [M] or NULL.
 * nthreads <= 0: OpenMP default. Returns 0, or -1 on bad arguments. */
int ffs_ref_sample_marginal(const double* U, int64_t L, int64_t N, int dtype, int64_t M, int64_t Np,
                            const double* uniforms, int32_t* positions, int32_t* flags, int nthreads)
{
    if (M == 0) return 0;
    if (check_args(U, L, N, dtype, Np) || !uniforms || !positions) return -1;
    size_t sb = scratch_bytes(L, N, Np, dtype);
    int bad = 0;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel num_threads(nthreads)
#endif
    {
        char* buf = (char*)malloc(sb);
        if (!buf) {
#ifdef _OPENMP
#pragma omp atomic write
#endif
            bad = 1;
        } else {
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 16)
#endif
            for (int64_t i = 0; i < M; ++i) {
                int f = run_one(U, L, N, dtype, Np, uniforms + i * 2 * Np, NULL, NULL,
                                positions + i * Np, NULL, NULL, NULL, buf);
                if (flags) flags[i] = f;
            }
            free(buf);
        }
    }
    return bad ? -2 : 0;
}

int ffs_ref_sample(const double* U, int64_t L, int64_t N, int dtype, int64_t M,
                   const double* uniforms, int32_t* positions, int32_t* flags, int nthreads)
{
    return ffs_ref_sample_marginal(U, L, N, dtype, M, N, uniforms, positions, flags, nthreads);
}

/* ffs_ref_weights: the first S samples of ffs_ref_sample_marginal, also returning the normalised
 * conditional weight vectors [S][Np][L] along the oracle's own path. */
int ffs_ref_weights(const double* U, int64_t L, int64_t N, int dtype, int64_t S, int64_t Np,
                    const double* uniforms, int32_t* positions, double* weights)
{
    if (S == 0) return 0;
    if (check_args(U, L, N, dtype, Np) || !uniforms || !positions || !weights) return -1;
    char* buf = (char*)malloc(scratch_bytes(L, N, Np, dtype));
    if (!buf) return -2;
    for (int64_t i = 0; i < S; ++i)
        run_one(U, L, N, dtype, Np, uniforms + i * 2 * Np, NULL, NULL, positions + i * Np,
                weights + i * Np * L, NULL, NULL, buf);
    free(buf);
    return 0;
}

/* ffs_ref_chain: teacher-forced chain for a given permutation m [N] and positions x [Np]:
 * weights [Np][L] normalised conditionals P(. | x_1..x_{k-1}; m), hnorm2 [Np] = |h'|^2 with
 * h'[k-1] = 1, totals [Np] = sum_x |u_x^T h|^2 with unit h (any may be NULL except weights). */
int ffs_ref_chain(const double* U, int64_t L, int64_t N, int dtype, int64_t Np, const int32_t* m,
                  const int32_t* x, double* weights, double* hnorm2, double* totals)
{
    if (check_args(U, L, N, dtype, Np) || !m || !x || !weights) return -1;
    char* buf = (char*)malloc(scratch_bytes(L, N, Np, dtype));
    if (!buf) return -2;
    int32_t* xo = (int32_t*)malloc(4 * (size_t)Np);
    int r = run_one(U, L, N, dtype, Np, NULL, m, x, xo, weights, hnorm2, totals, buf);
    free(xo);
    free(buf);
    return r;
}

/* ---------------------------------------------------------------- L-ensemble front end
 * PAPER.md:178-180 (text summarisation, step 2): the correlation matrix C = sum_j lambda_j u_j u_j^T
 * is eigendecomposed, "Each eigenvector u_j is selected with probability lambda_j/(lambda_j+1)",
 * and "The selected set of vectors ... form the matrix U in Eq. (1), according to which we perform
 * the fermion sampling with fermion particle number N" -- so each sample has its own N_i and U_i.
 *   V        : [L][K] eigenvectors (orthonormal columns), real or complex (dtype)
 *   lam      : [K] eigenvalues >= 0
 *   uniforms : [M][3K]: [0,K) keep draws (keep j iff u_j < lambda_j/(lambda_j+1), taken in fp64),
 *              [K,2K) the FFS permutation draws of U_i (first N_i used, reading Q6 with N = N_i),
 *              [2K,3K) the N_i selection draws (reading Q5)
 *   positions: [M][K] out, sampling order, entries k >= N_i set to -1; counts [M] = N_i; flags [M]
 * U_i = V[:, kept columns in ascending j] is built explicitly and sampled by run_one(). */
int ffs_ref_sample_lensemble(const double* V, const double* lam, int64_t L, int64_t K, int dtype, int64_t M,
                             const double* uniforms, int32_t* positions, int32_t* counts, int32_t* flags,
                             int nthreads)
{
    if (M == 0) return 0;
    if (!V || !lam || !uniforms || !positions || L < 1 || K < 1 || K > L) return -1;
    if (dtype != FFS_REF_F64 && dtype != FFS_REF_C128) return -1;
    size_t es = dtype == FFS_REF_C128 ? 16 : 8;
    size_t sb = scratch_bytes(L, K, K, dtype) + es * (size_t)(L * K) + 8 * (size_t)(2 * K) + 4 * (size_t)K + 64;
    int bad = 0;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel num_threads(nthreads)
#endif
    {
        char* buf = (char*)malloc(sb);
        if (!buf) {
#ifdef _OPENMP
#pragma omp atomic write
#endif
            bad = 1;
        } else {
            char* Ui = buf + scratch_bytes(L, K, K, dtype);
            double* row = (double*)(Ui + es * (size_t)(L * K));
            int32_t* kept = (int32_t*)(row + 2 * K);
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 16)
#endif
            for (int64_t i = 0; i < M; ++i) {
                const double* u = uniforms + i * 3 * K;
                int64_t n = 0;
                for (int64_t j = 0; j < K; ++j)
                    if (u[j] < lam[j] / (lam[j] + 1.0)) kept[n++] = (int32_t)j;
                for (int64_t k = 0; k < K; ++k) positions[i * K + k] = -1;
                if (counts) counts[i] = (int32_t)n;
                int f = 0;
                if (n > 0) {
                    for (int64_t x = 0; x < L; ++x)
                        for (int64_t c = 0; c < n; ++c)
                            memcpy(Ui + es * (size_t)(x * n + c), (const char*)V + es * (size_t)(x * K + kept[c]), es);
                    for (int64_t k = 0; k < n; ++k) {
                        row[k] = u[K + k];
                        row[n + k] = u[2 * K + k];
                    }
                    f = run_one((const double*)Ui, L, n, dtype, n, row, NULL, NULL, positions + i * K, NULL, NULL,
                                NULL, buf);
                }
                if (flags) flags[i] = f;
            }
            free(buf);
        }
    }
    return bad ? -2 : 0;
}

/* ---------------------------------------------------------------- observables of the samples
 * Occupation numbers <n_x> (SPEC.md:201 occupation oracle; "occupation number on
 * the site"), pair occupations <n_x n_y>, and the Slater-Jastrow / Gutzwiller reweighting of Supp S5
 * (PAPER.md:336-350): <O> = <J^2 o_L>_0 / <J^2>_0 with the Gutzwiller factor of Eq. 4
 * J(x) = exp(-V/2 sum_i n_{i,up} n_{i,down}), i.e. J^2 = exp(-V D), D = number of doubly occupied
 * sites. A spinful sample is a pair of independent FFS samples of the same U: rows 2s (up) and
 * 2s+1 (down) of positions (SPEC.md:387 N_up = N_down). Entries < 0 (L-ensemble padding) are
 * skipped. Plain loops over the samples, in sample order. */
int ffs_ref_occupation(const int32_t* positions, int64_t M, int64_t Np, int64_t L, uint64_t* occ)
{
    if (!positions || !occ || L < 1 || Np < 1 || M < 0) return -1;
    for (int64_t x = 0; x < L; ++x) occ[x] = 0;
    for (int64_t i = 0; i < M; ++i)
        for (int64_t k = 0; k < Np; ++k) {
            int32_t x = positions[i * Np + k];
            if (x >= 0 && x < L) occ[x] += 1;
        }
    return 0;
}

/* pair[x][y] = number of samples with both x and y occupied, x, y < W (the diagonal is <n_x>) */
int ffs_ref_pair_occupation(const int32_t* positions, int64_t M, int64_t Np, int64_t W, uint64_t* pair)
{
    if (!positions || !pair || W < 1 || Np < 1 || M < 0) return -1;
    for (int64_t q = 0; q < W * W; ++q) pair[q] = 0;
    for (int64_t i = 0; i < M; ++i)
        for (int64_t a = 0; a < Np; ++a) {
            int32_t x = positions[i * Np + a];
            if (x < 0 || x >= W) continue;
            for (int64_t b = 0; b < Np; ++b) {
                int32_t y = positions[i * Np + b];
                if (y >= 0 && y < W) pair[x * W + y] += 1;
            }
        }
    return 0;
}

/* result[0] = <J^2>_0 = (1/Ms) sum_s J_s^2; result[1] = <D>_J; result[2 + x] = <n_x>_J (both spins),
 * with <O>_J = sum_s J_s^2 O_s / sum_s J_s^2, Ms spinful samples. */
int ffs_ref_gutzwiller(const int32_t* positions, int64_t Ms, int64_t Np, int64_t L, double V, double* result)
{
    if (!positions || !result || L < 1 || Np < 1 || Ms < 1) return -1;
    char* up = (char*)calloc((size_t)L, 1);
    double* num = (double*)calloc((size_t)L, sizeof(double));
    if (!up || !num) { free(up); free(num); return -2; }
    double Z = 0.0, Dsum = 0.0;
    for (int64_t s = 0; s < Ms; ++s) {
        const int32_t* xu = positions + (2 * s) * Np;
        const int32_t* xd = positions + (2 * s + 1) * Np;
        for (int64_t k = 0; k < Np; ++k) if (xu[k] >= 0 && xu[k] < L) up[xu[k]] = 1;
        int64_t D = 0;
        for (int64_t k = 0; k < Np; ++k) if (xd[k] >= 0 && xd[k] < L && up[xd[k]]) ++D;
        const double J2 = exp(-V * (double)D);   /* J^2 = exp(2 * (-V/2) D) */
        Z += J2;
        Dsum += J2 * (double)D;
        for (int64_t k = 0; k < Np; ++k) {
            if (xu[k] >= 0 && xu[k] < L) num[xu[k]] += J2;
            if (xd[k] >= 0 && xd[k] < L) num[xd[k]] += J2;
        }
        for (int64_t k = 0; k < Np; ++k) if (xu[k] >= 0 && xu[k] < L) up[xu[k]] = 0;
    }
    result[0] = Z / (double)Ms;
    result[1] = Dsum / Z;
    for (int64_t x = 0; x < L; ++x) result[2 + x] = num[x] / Z;
    free(up);
    free(num);
    return 0;
}

/* ffs_ref_sample_metropolis: M samples of the Supp S7 variant (sample_metropolis above), Np steps,
 * Mc Metropolis updates per step. uniforms [M][Np + Np (1 + 2 Mc)], positions [M][Np], flags [M],
 * margins [M][Np] or NULL. */
int ffs_ref_sample_metropolis(const double* U, int64_t L, int64_t N, int dtype, int64_t M, int64_t Np, int64_t Mc,
                              const double* uniforms, int32_t* positions, int32_t* flags, double* margins,
                              int nthreads)
{
    if (M == 0) return 0;
    if (check_args(U, L, N, dtype, Np) || Mc < 0 || !uniforms || !positions) return -1;
    const int64_t stride = Np + Np * (1 + 2 * Mc);
    size_t sb = scratch_bytes(L, N, Np, dtype);
    int bad = 0;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel num_threads(nthreads)
#endif
    {
        char* buf = (char*)malloc(sb);
        if (!buf) {
#ifdef _OPENMP
#pragma omp atomic write
#endif
            bad = 1;
        } else {
            size_t es = dtype == FFS_REF_C128 ? 16 : 8;
            char* p = buf;
            void* R = p;      p += es * (size_t)(Np * Np);
            void* h = p;      p += es * (size_t)Np;
            p += 8 * (size_t)L;
            char* chosen = p; p += (size_t)L;
            int32_t* m = (int32_t*)(((uintptr_t)p + 3) & ~(uintptr_t)3);
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 16)
#endif
            for (int64_t i = 0; i < M; ++i) {
                const double* u = uniforms + i * stride;
                ffs_ref_permutation(u, N, Np, m);
                int f;
                if (dtype == FFS_REF_F64)
                    f = sample_metropolis_f64(U, L, N, Np, Mc, m, u, positions + i * Np,
                                              margins ? margins + i * Np : NULL, (double*)R, (double*)h, chosen);
                else
                    f = sample_metropolis_c128((const double _Complex*)U, L, N, Np, Mc, m, u, positions + i * Np,
                                               margins ? margins + i * Np : NULL, (double _Complex*)R,
                                               (double _Complex*)h, chosen);
                if (flags) flags[i] = f;
            }
            free(buf);
        }
    }
    return bad ? -2 : 0;
}

/* ffs_ref_sample_hkpv: M samples of the modified HKPV sampler (hkpv_chain above), Np steps.
 * uniforms [M][Np] selection draws; positions [M][Np]; flags [M]; weights [S][Np][L] and totals
 * [S][Np] of the first S samples (either may be NULL; S <= M). */
int ffs_ref_sample_hkpv(const double* U, int64_t L, int64_t N, int dtype, int64_t M, int64_t Np,
                        const double* uniforms, int32_t* positions, int32_t* flags, int64_t S, double* weights,
                        double* totals, int nthreads)
{
    if (M == 0) return 0;
    if (check_args(U, L, N, dtype, Np) || !uniforms || !positions || S < 0 || S > M) return -1;
    size_t es = dtype == FFS_REF_C128 ? 16 : 8;
    size_t sb = es * (size_t)(Np * N) + 8 * (size_t)L + (size_t)L + 64;
    int bad = 0;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel num_threads(nthreads)
#endif
    {
        char* buf = (char*)malloc(sb);
        if (!buf) {
#ifdef _OPENMP
#pragma omp atomic write
#endif
            bad = 1;
        } else {
            void* E = buf;
            double* r = (double*)(buf + es * (size_t)(Np * N));
            char* chosen = (char*)(r + L);
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 16)
#endif
            for (int64_t i = 0; i < M; ++i) {
                double* wt = (weights && i < S) ? weights + i * Np * L : NULL;
                double* tt = (totals && i < S) ? totals + i * Np : NULL;
                int f;
                if (dtype == FFS_REF_F64)
                    f = hkpv_chain_f64(U, L, N, Np, uniforms + i * Np, positions + i * Np, wt, tt, (double*)E, r,
                                       chosen);
                else
                    f = hkpv_chain_c128((const double _Complex*)U, L, N, Np, uniforms + i * Np, positions + i * Np,
                                        wt, tt, (double _Complex*)E, r, chosen);
                if (flags) flags[i] = f;
            }
            free(buf);
        }
    }
    return bad ? -2 : 0;
}

int ffs_ref_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
