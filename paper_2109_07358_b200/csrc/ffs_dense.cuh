// Lockstep-dense path for full sampling at large L (the C5 DPP-shaped workload): the candidate-
// weight contraction (a3) of S samples at the same block step runs as ONE dense FP64 GEMM on the
// tensor pipe (DMMA), instead of S per-sample gathered contractions that are bound by the
// bandwidth of the gathered U reads.
//
// For sample s at block start k0 (panel width B), the left-looking panel is
//   P_s = V_s[:, k0:k0+B] - V_s[:, 0:k0] W_s[0:k0, k0:k0+B],   V_s = U[:, m_s]
// = U Y_s with Y_s (N x B) the scatter of the coefficients into U's column space:
//   Y_s[m_j, c] = -W_s[j, k0+c] (j < k0),   Y_s[m_{k0+c}, c] = 1,   0 elsewhere.
// Stacking Y = [Y_0 .. Y_{S-1}] (N x S*B, row-major, row stride ldY), all S panels are
//   P = U Y   (L x N) (N x S*B)
// a plain dense GEMM whose A operand U is shared by every sample. It executes L*N*B FMAs per
// sample-block where the gathered form needs L*k0*B (2x over a full sample) but runs at the
// FP64 tensor-pipe rate instead of the ~2 flop/B of the gathered reads.
// The draws (a4), the rank-1 panel updates and the Gauss-Jordan update of W_s (a2/a5) run in
// ffs_cluster_kernel<..., STEP = true> (one cluster per sample, one block step per launch), which
// also scatters the next block's Y_s columns, so Y never needs re-zeroing: the nonzero rows of
// Y_s only grow ({m_j : j < k0+B}).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "ffs_kernel.cuh"

namespace ffsk {

// ---------------------------------------------------------------- DMMA DGEMM C = A B
// Row-major A [M][K] (lda), B [K][N] (ldb), C [M][N] (ldc); N % 128 == 0 and K % 2 == 0 (the
// host pads); rows >= M and k >= K are zero-filled. CTA tile 128 x 128 x 32, 8 warps as 4 (M) x 2
// (N), warp tile 32 x 64 = 4 x 8 DMMA m8n8k4 tiles, 3-stage cp.async pipeline of 32-deep K slices (192 KB smem).
constexpr int kGM = 128, kGN = 128, kGThreads = 256;
template <int kGK, int kGStages>
constexpr size_t gemm_smem() { return (size_t)kGStages * (kGM * kGK + kGK * kGN) * sizeof(double); }

struct DgemmParams {
  const double* A;
  const double* B;
  double* C;
  int64_t lda, ldb, ldc;
  int M, N, K;
  int panel;  // > 0: C in per-sample panel layout, column n -> C[(n / panel) * M * panel + row * panel + n % panel]
  // EPI = 1 (modified-HKPV residual update, ffs_hkpv.cuh): instead of storing C, subtract |C|^2
  // from the residuals r[sample][row] (row stride rld); real: column n is sample n; complex
  // (cplx = 1): columns 2s, 2s+1 are Re, Im of sample s; samples >= nsamp are padding
  double* r;
  int64_t rld;
  int nsamp, cplx;
};

__device__ __forceinline__ void dmma_884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc, int src_bytes) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(gsrc), "r"(src_bytes) : "memory");
}

// Shared-memory swizzles (8-byte element units): the A tile is [128][32] with element (r, c) at
// r*32 + (c ^ 4(r&3)); the B tile is [32][128] with (k, n) at k*128 + (n ^ 4(k&3)). The XOR only
// touches bits 2-3, so the 16-byte cp.async chunks stay contiguous, and each half-warp phase of
// the fragment loads (g = 0..3 or 4..7, t4 = 0..3) hits 16 distinct 8-byte bank slots.
// <32, 3>: 192 KB smem, 255 registers (fastest alone); <16, 4>: 128 KB, ~200 registers, which leaves
// room on each SM for a co-resident ffs_dense_gj_kernel CTA of the other half-batch (2-stream mode)
template <int kGK, int kGStages, int EPI = 0>
static __global__ void __launch_bounds__(kGThreads, 1) ffs_dgemm_kernel(const DgemmParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* As = reinterpret_cast<double*>(smem);
  double* Bs = As + kGStages * kGM * kGK;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int wm = warp & 3, wn = warp >> 2;
  const int g = lane >> 2, t4 = lane & 3;
  const int m0 = blockIdx.y * kGM, n0 = blockIdx.x * kGN;
  const int KT = (p.K + kGK - 1) / kGK;

  auto load_stage = [&](int st, int kt) {
    const int kk = kt * kGK;
    double* as = As + st * kGM * kGK;
    double* bs = Bs + st * kGK * kGN;
#pragma unroll
    for (int i = 0; i < kGM * kGK / 2 / kGThreads; ++i) {  // A: 128 rows x kGK/2 chunks
      const int c = t + i * kGThreads, r = c / (kGK / 2), ch = c % (kGK / 2);
      const int gr = m0 + r, gk = kk + 2 * ch;
      const bool in = gr < p.M && gk < p.K;
      const double* src = p.A + (in ? (size_t)gr * p.lda + gk : 0);
      cp_async16(as + r * kGK + ((2 * ch) ^ ((r & 3) << 2)), src, in ? 16 : 0);
    }
#pragma unroll
    for (int i = 0; i < kGK * kGN / 2 / kGThreads; ++i) {  // B: kGK rows x 64 chunks
      const int c = t + i * kGThreads, r = c >> 6, ch = c & 63;
      const int gk = kk + r;
      const bool in = gk < p.K;
      const double* src = p.B + (in ? (size_t)gk * p.ldb + n0 + 2 * ch : 0);
      cp_async16(bs + r * kGN + ((2 * ch) ^ ((r & 3) << 2)), src, in ? 16 : 0);
    }
  };

  double acc[4][8][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < kGStages - 1; ++s) {
    if (s < KT) load_stage(s, s);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int kt = 0; kt < KT; ++kt) {
    asm volatile("cp.async.wait_group %0;" ::"n"(kGStages - 2) : "memory");
    __syncthreads();
    {
      const int nk = kt + kGStages - 1;
      if (nk < KT) load_stage(nk % kGStages, nk);
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    const double* as = As + (kt % kGStages) * kGM * kGK + (wm * 32 + g) * kGK;
    const double* bs = Bs + (kt % kGStages) * kGK * kGN + t4 * kGN;
#pragma unroll
    for (int ks = 0; ks < kGK; ks += 4) {
      double a[4], b[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = as[i * 8 * kGK + ((ks + t4) ^ ((g & 3) << 2))];
#pragma unroll
      for (int j = 0; j < 8; ++j) b[j] = bs[ks * kGN + ((wn * 64 + j * 8 + g) ^ (t4 << 2))];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) dmma_884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if constexpr (EPI == 1) {
    // |C|^2 of the tile staged transposed in shared memory ([sample][row], row stride 129), then
    // subtracted from r with each column's rows contiguous across the threads (coalesced)
    static_assert(kGStages * (kGM * kGK + kGK * kGN) >= kGN * (kGM + 1), "staging tile fits the pipeline buffers");
    __syncthreads();
    double* Ts = reinterpret_cast<double*>(smem);
    constexpr int kLd = kGM + 1;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int rl = wm * 32 + i * 8 + g;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int cl = wn * 64 + j * 8 + 2 * t4;
        const double a = acc[i][j][0], b = acc[i][j][1];
        if (p.cplx) {
          Ts[(cl >> 1) * kLd + rl] = fma(a, a, b * b);
        } else {
          Ts[cl * kLd + rl] = a * a;
          Ts[(cl + 1) * kLd + rl] = b * b;
        }
      }
    }
    __syncthreads();
    const int ns = p.cplx ? kGN / 2 : kGN;
    const int s0 = p.cplx ? n0 / 2 : n0;
    for (int idx = t; idx < ns * kGM; idx += kGThreads) {
      const int sl = idx / kGM, rl = idx % kGM;
      const int row = m0 + rl, smp = s0 + sl;
      if (row < p.M && smp < p.nsamp) p.r[(size_t)smp * p.rld + row] -= Ts[sl * kLd + rl];
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + wm * 32 + i * 8 + g;
    if (row < p.M) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int col = n0 + wn * 64 + j * 8 + 2 * t4;
        const size_t off = p.panel > 0 ? (size_t)(col / p.panel) * p.M * p.panel + (size_t)row * p.panel + col % p.panel
                                       : (size_t)row * p.ldc + col;
        *reinterpret_cast<double2*>(p.C + off) = make_double2(acc[i][j][0], acc[i][j][1]);
      }
    }
  }
}

// Y for the first block: Y[m_c][s*B + c] = 1 (c < min(B, N')); Y is zero otherwise (memset).
// Complex T: Y is stored as its real 2N x 2ldY expansion (see dense_y_store).
template <typename T>
__device__ __forceinline__ void dense_y_store(double* Y, int64_t ldY, int n, int64_t col, T v);
template <>
__device__ __forceinline__ void dense_y_store<double>(double* Y, int64_t ldY, int n, int64_t col, double v) {
  Y[(size_t)n * ldY + col] = v;
}
// complex y at (n, col) -> real 2x2 block [[re, im], [-im, re]] at rows 2n, 2n+1, columns 2col, 2col+1
// of the real (2N x 2ldY) matrix, so that the real GEMM of U viewed as L x 2N (interleaved re, im)
// with it yields P interleaved: P'[x][2c] = sum Ur yr - Ui yi, P'[x][2c+1] = sum Ur yi + Ui yr.
template <>
__device__ __forceinline__ void dense_y_store<cplx>(double* Y, int64_t ldY, int n, int64_t col, cplx v) {
  double* r0 = Y + (size_t)(2 * n) * (2 * ldY) + 2 * col;
  double* r1 = r0 + 2 * ldY;
  *reinterpret_cast<double2*>(r0) = make_double2(v.re, v.im);
  *reinterpret_cast<double2*>(r1) = make_double2(-v.im, v.re);
}

template <typename T, int B>
static __global__ void ffs_dense_y0_kernel(const int32_t* __restrict__ perm, double* __restrict__ Y, int64_t ldY,
                                           int64_t base, int Sb, int Np) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= Sb * B) return;
  const int s = idx / B, c = idx % B;
  if (c < Np) dense_y_store<T>(Y, ldY, perm[(base + s) * Np + c], (int64_t)s * B + c, Sc<T>::one());
}

// ---------------------------------------------------------------- batched Gauss-Jordan update
// After the draws of block [k0, k0+B) of every batch sample (all samples share k0): with
// X_new = x_{k0..k0+B-1}, S = L U the B x B Schur block of the draws (pivot rows `Row`, inverse
// pivots `Pinv`), and j >= k1 = k0+B the later columns,
//   (1) Z[:, j] = V[X_new, j] - V[X_new, 0:k0] W[0:k0, j]
//   (2) Z[:, j] <- S^{-1} Z[:, j]
//   (3) W[0:k0, j] -= W[0:k0, k0:k1] Z[:, j],   W[k0:k1, j] = Z[:, j]
// then the next block's Y_s columns are scattered from W[0:k1, k1:k1+B] (tile 0 only).
// Grid (column tiles of TJ, batch samples); 4*TJ threads = TJ columns x 4 slices of i. W[0:k0, k0:k1]
// (the same B scalars for every column of a row) is read from global memory (L1 broadcast).

struct DenseGjParams {
  const double* U;          // [L][N]
  const int32_t* perm;      // [M][Np]
  const int32_t* positions; // [M][Np]
  const double* rowg;       // [Sb][B*B + B]
  double* W;                // [Sb][Np][Np]
  double* Y;                // [N][ldY] (complex: the real 2N x 2ldY expansion)
  int64_t ldY, base;        // ldY in scalars of T
  int N, Np, k0;
  int jend;                 // columns k1 <= j < jend are updated (Np: all later columns; k1 + B: only the
                            // next block's, when the rest follows in ffs_dense_gj2_kernel)
};

template <typename T, int B, int kGjTJ, int PARTS = 4>
__host__ __device__ inline size_t dense_gj_smem(int k0) {
  return sizeof(T) * ((size_t)B * k0 + PARTS * B * kGjTJ + B * kGjTJ + B * B + B) + sizeof(int) * 2 * B;
}

// CPT adjacent columns per thread (2 for real: 16-byte W accesses), 256 / PARTS column threads x
// PARTS slices of i per CTA of 256 threads (kGjTJ = 256 / PARTS * CPT columns); the i loops keep UNR
// independent W loads in flight per thread. PARTS = 4 for wide updates; PARTS = 64 (8 columns per
// CTA) for the 8-column updates of the paired schedule, where 4 slices left 16 threads walking k0 / 4
// rows each (0.21 ms per launch at k0 ~ 500).
template <typename T, int B, int kGjTJ, int PARTS = 4>
static __global__ void __launch_bounds__(256) ffs_dense_gj_kernel(const DenseGjParams q) {
  using S = Sc<T>;
  constexpr int CT = 256 / PARTS;  // column threads
  constexpr int CPT = kGjTJ / CT;
  constexpr int UNR = 8;
  static_assert(CPT == 1 || (CPT == 2 && sizeof(T) == 8), "two columns per thread only for real");
  extern __shared__ __align__(16) unsigned char smem[];
  const int k0 = q.k0, k1 = k0 + B, Np = q.Np, N = q.N;
  const int sl = blockIdx.y;
  const int64_t i_s = q.base + sl;
  const int t = threadIdx.x, jg = t % CT, part = t / CT;
  const int jl = jg * CPT;                        // first column of this thread within the tile
  const int j = k1 + blockIdx.x * kGjTJ + jl;     // first global column
  const int jend = q.jend;
  const bool has = j < jend;
  T* Vn = reinterpret_cast<T*>(smem);   // [k0][B]   V[X_new, 0:k0] transposed (a row's B values contiguous)
  T* Zp = Vn + (size_t)B * k0;          // [4][B][TJ] partial sums (negated)
  T* Zs = Zp + PARTS * B * kGjTJ;       // [B][TJ]
  T* RP = Zs + B * kGjTJ;               // Row [B][B], Pinv [B]
  int* xn = reinterpret_cast<int*>(RP + B * B + B);
  const int32_t* pm = q.perm + i_s * Np;
  const T* Ug = reinterpret_cast<const T*>(q.U);
  T* W = reinterpret_cast<T*>(q.W) + (size_t)sl * Np * Np;
  if (t < B) xn[t] = q.positions[i_s * Np + k0 + t];
  if (t < B * B + B) RP[t] = reinterpret_cast<const T*>(q.rowg)[(size_t)sl * (B * B + B) + t];
  __syncthreads();
  // gathers in batches of 8 independent loads per thread (one latency per batch, not per element)
  auto stage = [&](T* dst, int n, auto&& src) {
    for (int b0 = t; b0 < n; b0 += 8 * (int)blockDim.x) {
      T v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int idx = b0 + u * (int)blockDim.x;
        if (idx < n) v[u] = src(idx);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int idx = b0 + u * (int)blockDim.x;
        if (idx < n) dst[idx] = v[u];
      }
    }
  };
  stage(Vn, B * k0, [&](int idx) { return Ug[(size_t)xn[idx % B] * N + pm[idx / B]]; });
  __syncthreads();
  // 16-byte W accesses only when every row start is 16-byte aligned (N' even); the pair of
  // columns j, j+1 is loaded element-wise otherwise, and a pair past N' keeps its second slot 0
  const bool two = j + 1 < jend;
  const bool vec = two && (Np & 1) == 0;
  auto ldw = [&](int ii, T (&w)[CPT]) {
    const T* src = W + (size_t)ii * Np + j;
    if constexpr (CPT == 2) {
      if (vec) {
        const double2 v = *reinterpret_cast<const double2*>(src);
        w[0] = v.x;
        w[1] = v.y;
      } else {
        w[0] = src[0];
        w[1] = two ? src[1] : S::zero();
      }
    } else {
      w[0] = src[0];
    }
  };
  // (1) partial sums over this thread's slice of i
  T acc[CPT][B];  // minus the partial sums
#pragma unroll
  for (int e = 0; e < CPT; ++e)
#pragma unroll
    for (int tt = 0; tt < B; ++tt) acc[e][tt] = S::zero();
  if (has) {
    int ii = part;
    for (; ii + PARTS * (UNR - 1) < k0; ii += PARTS * UNR) {
      T w[UNR][CPT];
#pragma unroll
      for (int u = 0; u < UNR; ++u) ldw(ii + PARTS * u, w[u]);
#pragma unroll
      for (int u = 0; u < UNR; ++u)
#pragma unroll
        for (int tt = 0; tt < B; ++tt) {
          const T vn = Vn[(ii + PARTS * u) * B + tt];
#pragma unroll
          for (int e = 0; e < CPT; ++e) acc[e][tt] = S::fms(vn, w[u][e], acc[e][tt]);
        }
    }
    for (; ii < k0; ii += PARTS) {
      T w[CPT];
      ldw(ii, w);
#pragma unroll
      for (int tt = 0; tt < B; ++tt)
#pragma unroll
        for (int e = 0; e < CPT; ++e) acc[e][tt] = S::fms(Vn[ii * B + tt], w[e], acc[e][tt]);
    }
  }
#pragma unroll
  for (int e = 0; e < CPT; ++e)
#pragma unroll
    for (int tt = 0; tt < B; ++tt) Zp[(part * B + tt) * kGjTJ + jl + e] = acc[e][tt];
  __syncthreads();
  // Vn is dead: stage Wb = W[0:k0, k0:k1] ([k0][B], the same size) in its place for step (3), whose
  // per-row reads of it would otherwise be one dependent L2 round trip per row
  T* Wb = Vn;
  stage(Wb, k0 * B, [&](int idx) { return W[(size_t)(idx / B) * Np + k0 + idx % B]; });
  // (2) one thread per column: Z = S^{-1} (V[X_new, j] - sum)
  if (t < kGjTJ && k1 + blockIdx.x * kGjTJ + t < jend) {
    const int c = t, jc = k1 + blockIdx.x * kGjTJ + c;
    T z[B];
#pragma unroll
    for (int tt = 0; tt < B; ++tt) {
      T a01 = S::zero(), a23 = S::zero();  // pairwise over the slices
#pragma unroll 4
      for (int pp = 0; pp < PARTS; pp += 4) {
        a01 = S::add(a01, S::add(Zp[((pp + 0) * B + tt) * kGjTJ + c], Zp[((pp + 1) * B + tt) * kGjTJ + c]));
        a23 = S::add(a23, S::add(Zp[((pp + 2) * B + tt) * kGjTJ + c], Zp[((pp + 3) * B + tt) * kGjTJ + c]));
      }
      z[tt] = S::add(Ug[(size_t)xn[tt] * N + pm[jc]], S::add(a01, a23));
    }
    const T* Row = RP;
    const T* Pinv = RP + B * B;
#pragma unroll
    for (int tt = 1; tt < B; ++tt)
#pragma unroll
      for (int s2 = 0; s2 < tt; ++s2) z[tt] = S::fms(S::mul(Row[tt * B + s2], Pinv[s2]), z[s2], z[tt]);
#pragma unroll
    for (int tt = B - 1; tt >= 0; --tt) {
#pragma unroll
      for (int s2 = tt + 1; s2 < B; ++s2) z[tt] = S::fms(Row[tt * B + s2], z[s2], z[tt]);
      z[tt] = S::mul(z[tt], Pinv[tt]);
    }
#pragma unroll
    for (int tt = 0; tt < B; ++tt) {
      Zs[tt * kGjTJ + c] = z[tt];
      W[(size_t)(k0 + tt) * Np + jc] = z[tt];
    }
  }
  __syncthreads();
  // (3) rank-B update of the earlier rows
  if (has) {
    T z[CPT][B];
#pragma unroll
    for (int e = 0; e < CPT; ++e)
#pragma unroll
      for (int tt = 0; tt < B; ++tt) z[e][tt] = Zs[tt * kGjTJ + jl + e];
    auto upd = [&](int ii, T (&a)[CPT]) {
      const T* wb = Wb + (size_t)ii * B;  // the same B scalars for every thread of the warp: broadcast
#pragma unroll
      for (int tt = 0; tt < B; ++tt) {
        const T wv = wb[tt];
#pragma unroll
        for (int e = 0; e < CPT; ++e) a[e] = S::fms(wv, z[e][tt], a[e]);
      }
      T* dst = W + (size_t)ii * Np + j;
      if constexpr (CPT == 2) {
        if (vec) {
          *reinterpret_cast<double2*>(dst) = make_double2(a[0], a[1]);
        } else {
          dst[0] = a[0];
          if (two) dst[1] = a[1];
        }
      } else {
        dst[0] = a[0];
      }
    };
    // rows part, part + 4, ... < k0 in REVERSE order: step (1) streamed them upwards, so the rows
    // it read last are the ones most likely still in L2 (forward order re-reads a working set larger
    // than L2 in LRU's worst order)
    int m = (k0 - part + PARTS - 1) / PARTS - 1;
    for (; m >= UNR - 1; m -= UNR) {
      T a[UNR][CPT];
#pragma unroll
      for (int u = 0; u < UNR; ++u) ldw(part + PARTS * (m - u), a[u]);
#pragma unroll
      for (int u = 0; u < UNR; ++u) upd(part + PARTS * (m - u), a[u]);
    }
    for (; m >= 0; --m) {
      T a[CPT];
      ldw(part + PARTS * m, a);
      upd(part + PARTS * m, a);
    }
  }
  // next block's Y_s columns (the tile holding columns k1 .. k1+B-1)
  if (blockIdx.x == 0 && q.Y != nullptr) {  // (no Y when every block is contracted gathered)
    __syncthreads();
    const int nb1 = min(B, Np - k1);
    const int64_t col0 = (int64_t)sl * B;
    for (int idx = t; idx < k1 * B; idx += blockDim.x) {
      const int ii = idx / B, c = idx % B;
      FFS_CHECK(pm[ii] >= 0 && pm[ii] < N);
      dense_y_store<T>(q.Y, q.ldY, pm[ii], col0 + c, c < nb1 ? S::neg(W[(size_t)ii * Np + k1 + c]) : S::zero());
    }
    if (t < nb1) dense_y_store<T>(q.Y, q.ldY, pm[k1 + t], col0 + t, S::one());
  }
}


// ---------------------------------------------------------------- paired Gauss-Jordan update
// Two consecutive blocks' trailing updates in ONE pass over W (half the W traffic of two
// ffs_dense_gj_kernel launches: the update is HBM-bound, 8 FMAs per element read twice and written
// once). Blocks e = [k0, k0+8) and o = [k0+8, k0+16) with drawn rows X1, X2 and Schur factors
// S1 = L1 U1, S2 = L2 U2 (rowg1, rowg2). After block e only its next 8 columns were updated (the
// single-block kernel restricted to one 8-column tile), so for the later columns j >= k0+16 W still
// holds the state W_old of block start k0, while W[0:k0, k0:k0+8] = Wb1 and W[0:k0+8, k0+8:k0+16] =
// Wb2 are the two blocks' own coefficient panels. With a1 = V[X1, 0:k0] W_old[0:k0, j] and
// a2 = V[X2, 0:k0] W_old[0:k0, j] (one pass, 16 accumulators per column):
//   z1 = S1^{-1} (V[X1, j] - a1)
//   z2 = S2^{-1} (V[X2, j] - a2 + (V[X2, 0:k0] Wb1) z1 - V[X2, k0:k0+8] z1)
//   W[0:k0, j] = W_old - Wb1[0:k0] z1 - Wb2[0:k0] z2     (second pass)
//   W[k0:k0+8, j] = z1 - Wb2[k0:k0+8] z2,   W[k0+8:k0+16, j] = z2
// -- the same arithmetic as two single-block updates in a different association. T21 = V[X2, 0:k0] Wb1
// (8 x 8) is formed per CTA from the staged operands. The tile holding columns k0+16 .. k0+23
// scatters the next block's Y_s columns.
struct DenseGj2Params {
  const double* U;
  const int32_t* perm;
  const int32_t* positions;
  const double* rowg1;      // [Sb][B*B + B] of block e
  const double* rowg2;      // of block o
  const double* t21;        // [Sb][B*B] T21 = V[X2, 0:k0] Wb1 (ffs_dense_t21_kernel)
  double* W;
  double* Y;
  int64_t ldY, base;
  int N, Np, k0;
};

// T21[r][c] = sum_{i<k0} V[X2[r], m_i] W[i][k0+c], one CTA of 256 threads per batch sample
// (thread = (r, c) x 4 slices of i)
template <typename T, int B>
static __global__ void __launch_bounds__(256) ffs_dense_t21_kernel(const double* __restrict__ U, const int32_t* __restrict__ perm,
                                                                  const int32_t* __restrict__ positions,
                                                                  const double* __restrict__ Wg, double* __restrict__ t21,
                                                                  int64_t base, int N, int Np, int k0) {
  using S = Sc<T>;
  static_assert(B * B * 4 == 256, "thread mapping");
  __shared__ double red[4][B * B][2];
  const int sl = blockIdx.x, t = threadIdx.x, e = t % (B * B), part = t / (B * B);
  const int r = e / B, c = e % B;
  const int64_t i_s = base + sl;
  const int32_t* pm = perm + i_s * Np;
  const T* Ug = reinterpret_cast<const T*>(U);
  const T* W = reinterpret_cast<const T*>(Wg) + (size_t)sl * Np * Np;
  const size_t xrow = (size_t)positions[i_s * Np + k0 + B + r] * N;
  T a = S::zero();
  int i = part;
  for (; i + 12 < k0; i += 16) {
    T v[4], w[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      v[u] = Ug[xrow + pm[i + 4 * u]];
      w[u] = W[(size_t)(i + 4 * u) * Np + k0 + c];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) a = S::fms(v[u], w[u], a);
  }
  for (; i < k0; i += 4) a = S::fms(Ug[xrow + pm[i]], W[(size_t)i * Np + k0 + c], a);
  const T m = S::neg(a);
  red[part][e][0] = reinterpret_cast<const double*>(&m)[0];
  red[part][e][1] = S::kDoubles == 2 ? reinterpret_cast<const double*>(&m)[S::kDoubles - 1] : 0.0;
  __syncthreads();
  if (part == 0) {
    double* out = t21 + ((size_t)sl * B * B + e) * S::kDoubles;
    out[0] = (red[0][e][0] + red[1][e][0]) + (red[2][e][0] + red[3][e][0]);
    if (S::kDoubles == 2) out[1] = (red[0][e][1] + red[1][e][1]) + (red[2][e][1] + red[3][e][1]);
  }
}

constexpr int kGj2KC = 128;  // rows of V[X1 u X2, .] / of the coefficient panels staged per chunk

template <typename T, int B, int kGjTJ>
__host__ __device__ inline size_t dense_gj2_smem(int) {
  // chunk [kGj2KC][2B], Zp [4][2B][TJ], Zs [2B][TJ], T21 + V2n + Wb2 rows k0..k0+B-1 ([B][B] each),
  // Row/Pinv x 2, positions
  return sizeof(T) * ((size_t)2 * B * kGj2KC + 4 * 2 * B * kGjTJ + 2 * B * kGjTJ + 3 * B * B + 2 * (B * B + B)) +
         sizeof(int) * 2 * B + 16;
}

template <typename T, int B, int kGjTJ>
static __global__ void __launch_bounds__(256, 2) ffs_dense_gj2_kernel(const DenseGj2Params q) {
  using S = Sc<T>;
  constexpr int CPT = kGjTJ / 64;
  constexpr int UNR = sizeof(T) == 8 ? 4 : 2;  // complex: 16 complex accumulators + 4 loads in flight spill at 128 registers
  constexpr int B2 = 2 * B;
  static_assert(CPT == 1 || (CPT == 2 && sizeof(T) == 8), "two columns per thread only for real");
  extern __shared__ __align__(16) unsigned char smem[];
  const int k0 = q.k0, k1 = k0 + B, k2 = k0 + B2, Np = q.Np, N = q.N;
  const int sl = blockIdx.y;
  const int64_t i_s = q.base + sl;
  const int t = threadIdx.x, jg = t % 64, part = t / 64;
  const int jl = jg * CPT;
  const int j = k2 + blockIdx.x * kGjTJ + jl;
  const bool has = j < Np;
  T* Ch = reinterpret_cast<T*>(smem);     // [kGj2KC][2B]: V[X1 u X2, m_i] (pass 1), W[i][k0:k2] (pass 2)
  T* Zp = Ch + (size_t)B2 * kGj2KC;       // [4][2B][TJ]
  T* Zs = Zp + 4 * B2 * kGjTJ;            // [2B][TJ]: z1 (rows 0..B-1), z2
  T* T21 = Zs + B2 * kGjTJ;               // [B][B]
  T* V2n = T21 + B * B;                   // [B][B] V[X2, m_{k0+c}]
  T* W2r = V2n + B * B;                   // [B][B] Wb2 rows k0 .. k0+B-1
  T* RP1 = W2r + B * B;                   // Row1 [B][B], Pinv1 [B]
  T* RP2 = RP1 + B * B + B;
  int* xn = reinterpret_cast<int*>(RP2 + B * B + B);  // X1 (0..B-1), X2 (B..2B-1)
  const int32_t* pm = q.perm + i_s * Np;
  const T* Ug = reinterpret_cast<const T*>(q.U);
  T* W = reinterpret_cast<T*>(q.W) + (size_t)sl * Np * Np;
  if (t < B2) xn[t] = q.positions[i_s * Np + k0 + t];
  if (t < B * B + B) {
    RP1[t] = reinterpret_cast<const T*>(q.rowg1)[(size_t)sl * (B * B + B) + t];
    RP2[t] = reinterpret_cast<const T*>(q.rowg2)[(size_t)sl * (B * B + B) + t];
  }
  __syncthreads();
  if (t < B * B) {
    V2n[t] = Ug[(size_t)xn[B + t / B] * N + pm[k0 + t % B]];
    W2r[t] = W[(size_t)(k0 + t / B) * Np + k1 + t % B];
    T21[t] = reinterpret_cast<const T*>(q.t21)[(size_t)sl * B * B + t];
  }
  // one chunk of kc rows x 2B values: 8 independent loads per thread in flight
  auto stage = [&](int n, auto&& src) {
    for (int b0 = t; b0 < n; b0 += 8 * (int)blockDim.x) {
      T v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int idx = b0 + u * (int)blockDim.x;
        if (idx < n) v[u] = src(idx);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int idx = b0 + u * (int)blockDim.x;
        if (idx < n) Ch[idx] = v[u];
      }
    }
  };
  const bool two = j + 1 < Np;
  const bool vec = two && (Np & 1) == 0;
  auto ldw = [&](int ii, T (&w)[CPT]) {
    const T* src = W + (size_t)ii * Np + j;
    if constexpr (CPT == 2) {
      if (vec) {
        const double2 v = *reinterpret_cast<const double2*>(src);
        w[0] = v.x;
        w[1] = v.y;
      } else {
        w[0] = src[0];
        w[1] = two ? src[1] : S::zero();
      }
    } else {
      w[0] = src[0];
    }
  };
  // (1) minus the partial sums a1, a2 over this thread's slice of i (rows part, part + 4, ..)
  T acc[CPT][B2];
#pragma unroll
  for (int e = 0; e < CPT; ++e)
#pragma unroll
    for (int tt = 0; tt < B2; ++tt) acc[e][tt] = S::zero();
  for (int c0 = 0; c0 < k0; c0 += kGj2KC) {
    const int kc = min(kGj2KC, k0 - c0);
    __syncthreads();
    stage(B2 * kc, [&](int idx) { return Ug[(size_t)xn[idx % B2] * N + pm[c0 + idx / B2]]; });
    __syncthreads();
    if (has) {
      int il = part;  // kGj2KC is a multiple of 4: the slices stay aligned across chunks
      for (; il + 4 * (UNR - 1) < kc; il += 4 * UNR) {
        T w[UNR][CPT];
#pragma unroll
        for (int u = 0; u < UNR; ++u) ldw(c0 + il + 4 * u, w[u]);
#pragma unroll
        for (int u = 0; u < UNR; ++u)
#pragma unroll
          for (int tt = 0; tt < B2; ++tt) {
            const T vn = Ch[(il + 4 * u) * B2 + tt];
#pragma unroll
            for (int e = 0; e < CPT; ++e) acc[e][tt] = S::fms(vn, w[u][e], acc[e][tt]);
          }
      }
      for (; il < kc; il += 4) {
        T w[CPT];
        ldw(c0 + il, w);
#pragma unroll
        for (int tt = 0; tt < B2; ++tt)
#pragma unroll
          for (int e = 0; e < CPT; ++e) acc[e][tt] = S::fms(Ch[il * B2 + tt], w[e], acc[e][tt]);
      }
    }
  }
#pragma unroll
  for (int e = 0; e < CPT; ++e)
#pragma unroll
    for (int tt = 0; tt < B2; ++tt) Zp[(part * B2 + tt) * kGjTJ + jl + e] = acc[e][tt];
  __syncthreads();
  // (2) one thread per column: z1, z2 and the 2B new rows
  if (t < kGjTJ && k2 + blockIdx.x * kGjTJ + t < Np) {
    const int c = t, jc = k2 + blockIdx.x * kGjTJ + c;
    auto solve = [&](T (&z)[B], const T* Row, const T* Pinv) {
#pragma unroll
      for (int tt = 1; tt < B; ++tt)
#pragma unroll
        for (int s2 = 0; s2 < tt; ++s2) z[tt] = S::fms(S::mul(Row[tt * B + s2], Pinv[s2]), z[s2], z[tt]);
#pragma unroll
      for (int tt = B - 1; tt >= 0; --tt) {
#pragma unroll
        for (int s2 = tt + 1; s2 < B; ++s2) z[tt] = S::fms(Row[tt * B + s2], z[s2], z[tt]);
        z[tt] = S::mul(z[tt], Pinv[tt]);
      }
    };
    T z1[B], z2[B];
#pragma unroll
    for (int tt = 0; tt < B; ++tt) {
      const T a01 = S::add(Zp[(0 * B2 + tt) * kGjTJ + c], Zp[(1 * B2 + tt) * kGjTJ + c]);
      const T a23 = S::add(Zp[(2 * B2 + tt) * kGjTJ + c], Zp[(3 * B2 + tt) * kGjTJ + c]);
      z1[tt] = S::add(Ug[(size_t)xn[tt] * N + pm[jc]], S::add(a01, a23));
      const T b01 = S::add(Zp[(0 * B2 + B + tt) * kGjTJ + c], Zp[(1 * B2 + B + tt) * kGjTJ + c]);
      const T b23 = S::add(Zp[(2 * B2 + B + tt) * kGjTJ + c], Zp[(3 * B2 + B + tt) * kGjTJ + c]);
      z2[tt] = S::add(Ug[(size_t)xn[B + tt] * N + pm[jc]], S::add(b01, b23));
    }
    solve(z1, RP1, RP1 + B * B);
    // r2 += T21 z1 - V[X2, k0:k1] z1   (T21 = V[X2, 0:k0] Wb1)
#pragma unroll
    for (int tt = 0; tt < B; ++tt)
#pragma unroll
      for (int cc = 0; cc < B; ++cc) {
        z2[tt] = S::fms(S::neg(T21[tt * B + cc]), z1[cc], z2[tt]);
        z2[tt] = S::fms(V2n[tt * B + cc], z1[cc], z2[tt]);
      }
    solve(z2, RP2, RP2 + B * B);
#pragma unroll
    for (int tt = 0; tt < B; ++tt) {
      Zs[tt * kGjTJ + c] = z1[tt];
      Zs[(B + tt) * kGjTJ + c] = z2[tt];
      T w1 = z1[tt];
#pragma unroll
      for (int cc = 0; cc < B; ++cc) w1 = S::fms(W2r[tt * B + cc], z2[cc], w1);
      W[(size_t)(k0 + tt) * Np + jc] = w1;
      W[(size_t)(k1 + tt) * Np + jc] = z2[tt];
    }
  }
  __syncthreads();
  // (3) rank-2B update of the earlier rows, chunks in REVERSE order (the rows pass 1 read last are
  // the ones most likely still in L2); Ch holds W[i][k0:k2] = (Wb1[i], Wb2[i])
  T z[CPT][B2];
#pragma unroll
  for (int e = 0; e < CPT; ++e)
#pragma unroll
    for (int tt = 0; tt < B2; ++tt) z[e][tt] = has ? Zs[tt * kGjTJ + jl + e] : S::zero();
  auto upd = [&](int ii, int il, T (&a)[CPT]) {
    const T* wb = Ch + (size_t)il * B2;
#pragma unroll
    for (int tt = 0; tt < B2; ++tt) {
      const T wv = wb[tt];
#pragma unroll
      for (int e = 0; e < CPT; ++e) a[e] = S::fms(wv, z[e][tt], a[e]);
    }
    T* dst = W + (size_t)ii * Np + j;
    if constexpr (CPT == 2) {
      if (vec) {
        *reinterpret_cast<double2*>(dst) = make_double2(a[0], a[1]);
      } else {
        dst[0] = a[0];
        if (two) dst[1] = a[1];
      }
    } else {
      dst[0] = a[0];
    }
  };
  const int nchunks = (k0 + kGj2KC - 1) / kGj2KC;
  for (int cb = nchunks - 1; cb >= 0; --cb) {
    const int c0 = cb * kGj2KC;
    const int kc = min(kGj2KC, k0 - c0);
    __syncthreads();
    stage(B2 * kc, [&](int idx) { return W[(size_t)(c0 + idx / B2) * Np + k0 + idx % B2]; });
    __syncthreads();
    if (has) {
      int m = ((kc - part + 3) >> 2) - 1;
      for (; m >= UNR - 1; m -= UNR) {
        T a[UNR][CPT];
#pragma unroll
        for (int u = 0; u < UNR; ++u) ldw(c0 + part + 4 * (m - u), a[u]);
#pragma unroll
        for (int u = 0; u < UNR; ++u) upd(c0 + part + 4 * (m - u), part + 4 * (m - u), a[u]);
      }
      for (; m >= 0; --m) {
        T a[CPT];
        ldw(c0 + part + 4 * m, a);
        upd(c0 + part + 4 * m, part + 4 * m, a);
      }
    }
  }
  // next block's Y_s columns (the tile holding columns k2 .. k2+B-1)
  if (blockIdx.x == 0 && q.Y != nullptr) {
    __syncthreads();
    const int nb1 = min(B, Np - k2);
    const int64_t col0 = (int64_t)sl * B;
    for (int idx = t; idx < k2 * B; idx += blockDim.x) {
      const int ii = idx / B, c = idx % B;
      dense_y_store<T>(q.Y, q.ldY, pm[ii], col0 + c, c < nb1 ? S::neg(W[(size_t)ii * Np + k2 + c]) : S::zero());
    }
    if (t < nb1) dense_y_store<T>(q.Y, q.ldY, pm[k2 + t], col0 + t, S::one());
  }
}


// ---------------------------------------------------------------- Ozaki-emulated FP64 GEMM
// P = U Y on the INT8 tensor cores (tcgen05.mma.kind::i8, TMEM accumulators). Rows of A (= U, or
// its real L x 2N view) and columns of B (= Y, or its real expansion) are scaled by powers of two
// (frexp: |x 2^-e| < 1) and split into NS signed 7-bit slices: x = 2^e sum_i q_i 2^{-7(i+1)}.
// The slice products A_i B_j with i + j < NS are exact in int32 (|q| <= 127; NS (K) 127^2 < 2^31
// for K <= 16384); the CTA keeps the NS partial sums D_d = sum_{i+j=d} A_i B_j of its 128 x 64
// tile in NS TMEM accumulators (NS x 64 <= 512 columns) and the epilogue forms
// 2^(ea + eb) sum_d 2^{-7(d+2)} D_d in fp64. The dropped terms (i + j >= NS) are below
// 2^-(7 NS) of the row/column scales: NS = 8 (the default) leaves a normwise panel error of
// <= 1.3e-15, the level of a native fp64 GEMM; NS = 7 leaves <= 2.2e-13 (tools/ozaki_floor.py,
// profiles/ozaki_floor_r01.txt).
// Operands reach shared memory by TMA (3-D tensor maps [NS][rows][Kp], 64-byte swizzle) issued
// by one thread; one thread issues the MMAs; full/empty mbarriers hand the two stages over.
constexpr int kOzMaxS = 8;
constexpr int kOzBM = 128, kOzBN = 64, kOzBK = 64, kOzStages = 2, kOzThreads = 320;  // 8 epilogue warps + TMA + MMA
constexpr int kOzTA = kOzBM * kOzBK, kOzTB = kOzBN * kOzBK;
template <int NS> constexpr int oz_stage_bytes() { return NS * (kOzTA + kOzTB); }
template <int NS>
constexpr size_t oz_smem() { return (size_t)kOzStages * oz_stage_bytes<NS>() + (2 * kOzStages + 2) * 8 + 16 + 1024; }
static_assert(oz_smem<kOzMaxS>() <= 227 * 1024, "two stages of 8 slices fit shared memory");

struct OzakiParams {
  const int* ea;  // [M] row exponents of A
  const int* eb;  // [N] column exponents of B
  double* C;      // per-sample panel layout (see DgemmParams::panel)
  int M, N, K;    // K padded to a multiple of kOzBK (zero slices)
  int panel;
  // tile raster: consecutive CTAs share one operand tile and stream the other one, which must
  // stay L2-resident across the sweep. m_fast = 1: blockIdx.x walks the M-tiles (A streamed,
  // B tile shared; for B >> A, e.g. C4's 512 MB of Y slices vs 32 MB of U slices);
  // m_fast = 0: blockIdx.x walks the N-tiles (B streamed; C5: 64 MB of Y vs 128 MB of U)
  int m_fast;
};

__device__ __forceinline__ unsigned oz_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t oz_desc(const void* base) {  // K-major, 64-byte swizzle, SBO 512 B
  uint64_t d = (oz_u32(base) >> 4) & 0x3FFF;
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}
// descriptor of an operand `off` bytes past the one `base` describes: the start address (>> 4)
// is the low 14-bit field and shared memory is < 256 KB, so the offset adds to the low word
// without a carry (one uniform add per MMA instead of recomputing the descriptor)
__device__ __forceinline__ uint64_t oz_desc_add(uint64_t base, uint32_t off) {
  const uint32_t lo = (uint32_t)base + (off >> 4), hi = (uint32_t)(base >> 32);
  return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ void oz_mbar_init(uint64_t* b, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(oz_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void oz_mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "OW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra OW_%=;\n\t}" ::"r"(oz_u32(b)),
      "r"(parity)
      : "memory");
}

// Persistent: one CTA per SM walks the tiles t = blockIdx.x, blockIdx.x + gridDim.x, ... (the
// raster of OzakiParams::m_fast). TMEM is allocated and the barriers initialised once; the TMA
// producer streams the K chunks of consecutive tiles through the two stages without a break; the
// MMA issuer starts a tile as soon as the epilogue has drained the accumulators of the previous one
// (tmem_empty), and the epilogue's fp64 scaling and global stores overlap the next tile's MMAs.
template <int NS>
static __global__ void __launch_bounds__(kOzThreads, 1) ffs_ozaki_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                                                                            const __grid_constant__ CUtensorMap tmB,
                                                                            const OzakiParams p) {
  extern __shared__ __align__(1024) unsigned char oz_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(oz_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + kOzStages * oz_stage_bytes<NS>());
  uint64_t* empty = full + kOzStages;
  uint64_t* tfull = empty + kOzStages;  // MMA -> epilogue: the tile's accumulators are complete
  uint64_t* tempty = tfull + 1;         // epilogue -> MMA: the accumulators have been read
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int KT = p.K / kOzBK;
  const int mt = (p.M + kOzBM - 1) / kOzBM, nt = p.N / kOzBN;
  const int ntiles = mt * nt;
  auto tile_origin = [&](int tt, int& m0, int& n0) {
    const int a = p.m_fast ? tt % mt : tt / nt, b = p.m_fast ? tt / mt : tt % nt;
    m0 = a * kOzBM;
    n0 = b * kOzBN;
  };
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(oz_u32(tmem_slot)), "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (t == 0) {
    for (int s = 0; s < kOzStages; ++s) {
      oz_mbar_init(full + s, 1);
      oz_mbar_init(empty + s, 1);
    }
    oz_mbar_init(tfull, 1);
    oz_mbar_init(tempty, 256);  // the 8 epilogue warps
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  if (warp == 8 && lane == 0) {  // TMA producer
    int g = 0;                   // K chunks issued so far (all tiles)
    for (int tt = blockIdx.x; tt < ntiles; tt += gridDim.x) {
      int m0, n0;
      tile_origin(tt, m0, n0);
      for (int kt = 0; kt < KT; ++kt, ++g) {
        const int st = g % kOzStages;
        if (g >= kOzStages) oz_mbar_wait(empty + st, ((g / kOzStages) - 1) & 1);
        unsigned char* sb = sm + st * oz_stage_bytes<NS>();
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(oz_u32(full + st)),
                     "r"(oz_stage_bytes<NS>())
                     : "memory");
#pragma unroll
        for (int i = 0; i < NS; ++i) {
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                  oz_u32(sb + i * kOzTA)),
              "l"(&tmA), "r"(kt * kOzBK), "r"(m0), "r"(i), "r"(oz_u32(full + st))
              : "memory");
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                  oz_u32(sb + NS * kOzTA + i * kOzTB)),
              "l"(&tmB), "r"(kt * kOzBK), "r"(n0), "r"(i), "r"(oz_u32(full + st))
              : "memory");
        }
      }
    }
  } else if (warp == 9 && lane == 0) {  // MMA issuer
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kOzBN >> 3) << 17) | ((uint32_t)(kOzBM >> 4) << 24);
    int g = 0, it = 0;
    for (int tt = blockIdx.x; tt < ntiles; tt += gridDim.x, ++it) {
      if (it > 0) oz_mbar_wait(tempty, (it - 1) & 1);  // the previous tile's accumulators were read
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int kt = 0; kt < KT; ++kt, ++g) {
        const int st = g % kOzStages;
        oz_mbar_wait(full + st, (g / kOzStages) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const unsigned char* sb = sm + st * oz_stage_bytes<NS>();
        const uint64_t da0 = oz_desc(sb), db0 = oz_desc(sb + NS * kOzTA);
#pragma unroll
        for (int i = 0; i < NS; ++i)
#pragma unroll
          for (int j = 0; j < NS - i; ++j)
#pragma unroll
            for (int ks = 0; ks < kOzBK / 32; ++ks) {
              const uint64_t da = oz_desc_add(da0, i * kOzTA + ks * 32);
              const uint64_t db = oz_desc_add(db0, j * kOzTB + ks * 32);
              const uint32_t acc = (kt > 0 || ks > 0 || i > 0) ? 1u : 0u;  // first write of D_{i+j}: i = 0
              asm volatile(
                  "{\n\t.reg .pred p;\n\t"
                  "setp.ne.b32 p, %4, 0;\n\t"
                  "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + (uint32_t)((i + j) * kOzBN)),
                  "l"(da), "l"(db), "r"(idesc), "r"(acc)
                  : "memory");
            }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(oz_u32(empty + st))
                     : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(oz_u32(tfull))
                   : "memory");
    }
  }
  if (warp < 8) {  // epilogue: warp w reads TMEM lanes 32 (w % 4) .. (tile rows), columns 32 (w / 4) ..
    constexpr int kEC = kOzBN / 2;  // columns per epilogue warp
    const int q = warp & 3, ch = (warp >> 2) * kEC;
    int it = 0;
    for (int tt = blockIdx.x; tt < ntiles; tt += gridDim.x, ++it) {
      int m0, n0;
      tile_origin(tt, m0, n0);
      oz_mbar_wait(tfull, it & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      double acc[kEC];
#pragma unroll
      for (int c = 0; c < kEC; ++c) acc[c] = 0.0;
#pragma unroll
      for (int d = NS - 1; d >= 0; --d) {  // smallest terms first
        const double sc = ldexp(1.0, -7 * (d + 2));
        uint32_t v[32];
        const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(d * kOzBN + ch);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int c = 0; c < 32; ++c) acc[c] = fma((double)(int)v[c], sc, acc[c]);
      }
      // every accumulator of this tile is in registers: hand TMEM back to the MMA issuer
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(oz_u32(tempty)) : "memory");
      const int row = m0 + q * 32 + lane;
      if (row < p.M) {
        // 2^(ea + eb) as one multiply by an exact power of two built from its biased exponent
        // (ldexp outside the normal range); panel (8 or 16) is a power of two
        const int er = p.ea[row];
        const int lp = __ffs(p.panel) - 1;
        double* crow = p.C + (size_t)row * p.panel;
        const size_t sstride = (size_t)p.M * p.panel;
#pragma unroll
        for (int c = 0; c < kEC; c += 2) {
          const int col = n0 + ch + c;
          FFS_CHECK(col + 1 < p.N);
          const int2 e2 = *reinterpret_cast<const int2*>(p.eb + col);
          const int b0 = 1023 + er + e2.x, b1 = 1023 + er + e2.y;  // biased exponents
          const double s0 = (b0 > 0 && b0 < 2047) ? __longlong_as_double((long long)b0 << 52) : ldexp(1.0, er + e2.x);
          const double s1 = (b1 > 0 && b1 < 2047) ? __longlong_as_double((long long)b1 << 52) : ldexp(1.0, er + e2.y);
          *reinterpret_cast<double2*>(crow + (size_t)(col >> lp) * sstride + (col & (p.panel - 1))) =
              make_double2(acc[c] * s0, acc[c + 1] * s1);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
}

// ---- 2-SM variant (tcgen05 cta_group::2): a cluster of two CTAs on one TPC computes a 256 x 64
// tile. Each CTA loads its 128 rows of the A slices and HALF (32 columns) of the B slices; the
// leader CTA issues M = 256 MMAs that read A from each CTA's own shared memory and B from both,
// writing rows 0-127 to the leader's TMEM and 128-255 to the peer's. Per SM and K chunk that is
// 80 KB of TMA loads and 5 KB of shared-memory operand reads per MMA instead of 96 KB / 6 KB for
// the one-SM tile, at the same MMA count (B300_MICROARCH: one-SM MMA with both operands in shared
// memory is limited by the operand reads). Barriers: the leader's full barrier expects both CTAs'
// bytes (both CTAs' TMA loads signal it); the leader's MMA commits release the stage and the
// accumulators in both CTAs; both CTAs' epilogues hand the TMEM back to the leader.
constexpr int kOz2TB = (kOzBN / 2) * kOzBK;  // one CTA's half of the B tile (32 columns)
template <int NS> constexpr int oz2_stage_bytes() { return NS * (kOzTA + kOz2TB); }
template <int NS>
constexpr size_t oz2_smem() { return (size_t)kOzStages * oz2_stage_bytes<NS>() + (2 * kOzStages + 2) * 8 + 16 + 1024; }

__device__ __forceinline__ unsigned oz2_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void oz2_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int NS>
static __global__ void __launch_bounds__(kOzThreads, 1) ffs_ozaki_gemm2_kernel(const __grid_constant__ CUtensorMap tmA,
                                                                             const __grid_constant__ CUtensorMap tmB,
                                                                             const OzakiParams p) {
  extern __shared__ __align__(1024) unsigned char oz_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(oz_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + kOzStages * oz2_stage_bytes<NS>());
  uint64_t* empty = full + kOzStages;
  uint64_t* tfull = empty + kOzStages;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const unsigned crank = oz2_rank();
  const bool leader = crank == 0;
  const int KT = p.K / kOzBK;
  const int mt = (p.M + 2 * kOzBM - 1) / (2 * kOzBM), nt = p.N / kOzBN;  // pair tiles: 256 x 64
  const int ntiles = mt * nt;
  const int pfirst = (int)(blockIdx.x >> 1), pstep = (int)(gridDim.x >> 1);
  auto tile_origin = [&](int tt, int& m0, int& n0) {  // this CTA's 128 rows of the pair tile
    const int a = p.m_fast ? tt % mt : tt / nt, b = p.m_fast ? tt / mt : tt % nt;
    m0 = a * 2 * kOzBM + (int)crank * kOzBM;
    n0 = b * kOzBN;
  };
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(oz_u32(tmem_slot)), "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  if (t == 0) {
    for (int s = 0; s < kOzStages; ++s) {
      oz_mbar_init(full + s, 1);
      oz_mbar_init(empty + s, 1);
    }
    oz_mbar_init(tfull, 1);
    oz_mbar_init(tempty, 2 * 256);  // both CTAs' epilogue threads
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  oz2_cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t kPeerMask = 0xFEFFFFFFu;  // shared::cluster address of the leader's copy
  if (warp == 8 && lane == 0) {  // TMA producer (both CTAs)
    int g = 0;
    for (int tt = pfirst; tt < ntiles; tt += pstep) {
      int m0, n0;
      tile_origin(tt, m0, n0);
      const int nb0 = n0 + (int)crank * (kOzBN / 2);
      for (int kt = 0; kt < KT; ++kt, ++g) {
        const int st = g % kOzStages;
        if (g >= kOzStages) oz_mbar_wait(empty + st, ((g / kOzStages) - 1) & 1);
        unsigned char* sb = sm + st * oz2_stage_bytes<NS>();
        const uint32_t fb = oz_u32(full + st) & kPeerMask;
        if (leader)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(oz_u32(full + st)),
                       "r"(2 * oz2_stage_bytes<NS>())
                       : "memory");
#pragma unroll
        for (int i = 0; i < NS; ++i) {
          asm volatile(
              "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                  oz_u32(sb + i * kOzTA)),
              "l"(&tmA), "r"(kt * kOzBK), "r"(m0), "r"(i), "r"(fb)
              : "memory");
          asm volatile(
              "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                  oz_u32(sb + NS * kOzTA + i * kOz2TB)),
              "l"(&tmB), "r"(kt * kOzBK), "r"(nb0), "r"(i), "r"(fb)
              : "memory");
        }
      }
    }
  } else if (warp == 9 && lane == 0 && leader) {  // MMA issuer: the leader CTA only
    const uint32_t idesc =
        (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kOzBN >> 3) << 17) | ((uint32_t)((2 * kOzBM) >> 4) << 24);
    const uint16_t mask = 0x3;
    int g = 0, it = 0;
    for (int tt = pfirst; tt < ntiles; tt += pstep, ++it) {
      if (it > 0) oz_mbar_wait(tempty, (it - 1) & 1);  // both CTAs read the previous accumulators
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int kt = 0; kt < KT; ++kt, ++g) {
        const int st = g % kOzStages;
        oz_mbar_wait(full + st, (g / kOzStages) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const unsigned char* sb = sm + st * oz2_stage_bytes<NS>();
        const uint64_t da0 = oz_desc(sb), db0 = oz_desc(sb + NS * kOzTA);
#pragma unroll
        for (int i = 0; i < NS; ++i)
#pragma unroll
          for (int j = 0; j < NS - i; ++j)
#pragma unroll
            for (int ks = 0; ks < kOzBK / 32; ++ks) {
              const uint64_t da = oz_desc_add(da0, i * kOzTA + ks * 32);
              const uint64_t db = oz_desc_add(db0, j * kOz2TB + ks * 32);
              const uint32_t acc = (kt > 0 || ks > 0 || i > 0) ? 1u : 0u;
              asm volatile(
                  "{\n\t.reg .pred p;\n\t"
                  "setp.ne.b32 p, %4, 0;\n\t"
                  "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + (uint32_t)((i + j) * kOzBN)),
                  "l"(da), "l"(db), "r"(idesc), "r"(acc)
                  : "memory");
            }
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                         oz_u32(empty + st)),
                     "h"(mask)
                     : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                       oz_u32(tfull)),
                   "h"(mask)
                   : "memory");
    }
  }
  if (warp < 8) {  // epilogue (both CTAs): this CTA's 128 rows of the pair tile
    constexpr int kEC = kOzBN / 2;
    const int q = warp & 3, ch = (warp >> 2) * kEC;
    const uint32_t te = oz_u32(tempty) & kPeerMask;
    int it = 0;
    for (int tt = pfirst; tt < ntiles; tt += pstep, ++it) {
      int m0, n0;
      tile_origin(tt, m0, n0);
      oz_mbar_wait(tfull, it & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      double acc[kEC];
#pragma unroll
      for (int c = 0; c < kEC; ++c) acc[c] = 0.0;
#pragma unroll
      for (int d = NS - 1; d >= 0; --d) {
        const double sc = ldexp(1.0, -7 * (d + 2));
        uint32_t v[32];
        const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(d * kOzBN + ch);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int c = 0; c < 32; ++c) acc[c] = fma((double)(int)v[c], sc, acc[c]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(te) : "memory");
      const int row = m0 + q * 32 + lane;
      if (row < p.M) {
        const int er = p.ea[row];
        const int lp = __ffs(p.panel) - 1;
        double* crow = p.C + (size_t)row * p.panel;
        const size_t sstride = (size_t)p.M * p.panel;
#pragma unroll
        for (int c = 0; c < kEC; c += 2) {
          const int col = n0 + ch + c;
          FFS_CHECK(col + 1 < p.N);
          const int2 e2 = *reinterpret_cast<const int2*>(p.eb + col);
          const int b0 = 1023 + er + e2.x, b1 = 1023 + er + e2.y;
          const double s0 = (b0 > 0 && b0 < 2047) ? __longlong_as_double((long long)b0 << 52) : ldexp(1.0, er + e2.x);
          const double s1 = (b1 > 0 && b1 < 2047) ? __longlong_as_double((long long)b1 << 52) : ldexp(1.0, er + e2.y);
          *reinterpret_cast<double2*>(crow + (size_t)(col >> lp) * sstride + (col & (p.panel - 1))) =
              make_double2(acc[c] * s0, acc[c + 1] * s1);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  oz2_cluster_sync();  // neither CTA leaves while the other may still signal it or read its TMEM
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
}

// ---- wide 2-SM variant: 256 x 128 pair tiles in TWO PASSES of four diagonals each.
// With N = 64 every MMA reads 4 KB of A and 2 KB of B from shared memory for 32 tensor-pipe cycles
// (192 B/clk against the ~128 B/clk the tensor core can read: the INT8 pipe cannot exceed ~67 %,
// measured 59.7 %, profiles/r02/final/full_ozaki2_dpp_raw.csv). Eight accumulators of 128 columns do
// not fit TMEM (512 columns), so a tile runs as two "virtual tiles": pass 1 accumulates the
// diagonals d = i + j = 4..7 (26 slice products, all 8 slices of both operands), pass 0 the
// diagonals 0..3 (10 products, slices 0..3 only); each pass has four 128-column accumulators and
// its MMAs read 4 KB + 4 KB per 64 cycles. Pass 1 (the small terms) stores its scaled sum, pass 0
// adds its own to it (the tile is L2-resident between the two). Same TMA / MMA / epilogue roles and
// barrier protocol as ffs_ozaki_gemm2_kernel, one K loop per virtual tile; the stage holds 8 A
// slices (8 KB each) and 8 half B slices (64 columns, 4 KB each).
constexpr int kOzWBN = 128;
constexpr int kOzWTB = (kOzWBN / 2) * kOzBK;  // one CTA's half of a B slice tile (64 columns)
constexpr int oz2w_stage_bytes() { return kOzMaxS * (kOzTA + kOzWTB); }
constexpr size_t oz2w_smem() { return (size_t)kOzStages * oz2w_stage_bytes() + (2 * kOzStages + 2) * 8 + 16 + 1024; }
static_assert(oz2w_smem() <= 227 * 1024, "two stages of the wide tile fit shared memory");

static __global__ void __launch_bounds__(kOzThreads, 1) ffs_ozaki_gemm2w_kernel(const __grid_constant__ CUtensorMap tmA,
                                                                              const __grid_constant__ CUtensorMap tmB,
                                                                              const OzakiParams p) {
  constexpr int NS = 8;
  extern __shared__ __align__(1024) unsigned char oz_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(oz_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + kOzStages * oz2w_stage_bytes());
  uint64_t* empty = full + kOzStages;
  uint64_t* tfull = empty + kOzStages;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const unsigned crank = oz2_rank();
  const bool leader = crank == 0;
  const int KT = p.K / kOzBK;
  const int mt = (p.M + 2 * kOzBM - 1) / (2 * kOzBM), nt = p.N / kOzWBN;  // pair tiles: 256 x 128
  const int ntiles = mt * nt;
  const int pfirst = (int)(blockIdx.x >> 1), pstep = (int)(gridDim.x >> 1);
  auto tile_origin = [&](int tt, int& m0, int& n0) {  // this CTA's 128 rows of the pair tile
    const int a = p.m_fast ? tt % mt : tt / nt, b = p.m_fast ? tt / mt : tt % nt;
    m0 = a * 2 * kOzBM + (int)crank * kOzBM;
    n0 = b * kOzWBN;
  };
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(oz_u32(tmem_slot)), "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  if (t == 0) {
    for (int s = 0; s < kOzStages; ++s) {
      oz_mbar_init(full + s, 1);
      oz_mbar_init(empty + s, 1);
    }
    oz_mbar_init(tfull, 1);
    oz_mbar_init(tempty, 2 * 256);  // both CTAs' epilogue threads
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  oz2_cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t kPeerMask = 0xFEFFFFFFu;  // shared::cluster address of the leader's copy
  // virtual tiles: (tile, pass) with pass 1 (diagonals 4..7) first, then pass 0 (diagonals 0..3)
  if (warp == 8 && lane == 0) {  // TMA producer (both CTAs)
    int g = 0;
    for (int tt = pfirst; tt < ntiles; tt += pstep) {
      int m0, n0;
      tile_origin(tt, m0, n0);
      const int nb0 = n0 + (int)crank * (kOzWBN / 2);
      for (int pass = 1; pass >= 0; --pass) {
        const int nsl = pass ? NS : NS / 2;  // slices this pass reads
        for (int kt = 0; kt < KT; ++kt, ++g) {
          const int st = g % kOzStages;
          if (g >= kOzStages) oz_mbar_wait(empty + st, ((g / kOzStages) - 1) & 1);
          unsigned char* sb = sm + st * oz2w_stage_bytes();
          const uint32_t fb = oz_u32(full + st) & kPeerMask;
          if (leader)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(oz_u32(full + st)),
                         "r"(2 * nsl * (kOzTA + kOzWTB))
                         : "memory");
          for (int i = 0; i < nsl; ++i) {
            asm volatile(
                "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                    oz_u32(sb + i * kOzTA)),
                "l"(&tmA), "r"(kt * kOzBK), "r"(m0), "r"(i), "r"(fb)
                : "memory");
            asm volatile(
                "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                    oz_u32(sb + NS * kOzTA + i * kOzWTB)),
                "l"(&tmB), "r"(kt * kOzBK), "r"(nb0), "r"(i), "r"(fb)
                : "memory");
          }
        }
      }
    }
  } else if (warp == 9 && lane == 0 && leader) {  // MMA issuer: the leader CTA only
    const uint32_t idesc =
        (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kOzWBN >> 3) << 17) | ((uint32_t)((2 * kOzBM) >> 4) << 24);
    const uint16_t mask = 0x3;
    int g = 0, it = 0;
    for (int tt = pfirst; tt < ntiles; tt += pstep) {
      for (int pass = 1; pass >= 0; --pass, ++it) {
        if (it > 0) oz_mbar_wait(tempty, (it - 1) & 1);  // both CTAs read the previous accumulators
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int dmin = pass ? NS / 2 : 0;
        for (int kt = 0; kt < KT; ++kt, ++g) {
          const int st = g % kOzStages;
          oz_mbar_wait(full + st, (g / kOzStages) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const unsigned char* sb = sm + st * oz2w_stage_bytes();
          const uint64_t da0 = oz_desc(sb), db0 = oz_desc(sb + NS * kOzTA);
#pragma unroll
          for (int i = 0; i < NS; ++i)
#pragma unroll
            for (int j = 0; j < NS - i; ++j) {
              const int d = i + j;
              if (d < dmin || d >= dmin + NS / 2) continue;
#pragma unroll
              for (int ks = 0; ks < kOzBK / 32; ++ks) {
                const uint64_t da = oz_desc_add(da0, i * kOzTA + ks * 32);
                const uint64_t db = oz_desc_add(db0, j * kOzWTB + ks * 32);
                const uint32_t acc = (kt > 0 || ks > 0 || i > 0) ? 1u : 0u;  // first write of D_d: i = 0
                asm volatile(
                    "{\n\t.reg .pred p;\n\t"
                    "setp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + (uint32_t)((d - dmin) * kOzWBN)),
                    "l"(da), "l"(db), "r"(idesc), "r"(acc)
                    : "memory");
              }
            }
          asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                           oz_u32(empty + st)),
                       "h"(mask)
                       : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                         oz_u32(tfull)),
                     "h"(mask)
                     : "memory");
      }
    }
  }
  if (warp < 8) {  // epilogue (both CTAs): warp w: rows 32 (w % 4) .., columns 64 (w / 4) .. of this CTA's 128 x 128
    const int q = warp & 3, ch0 = (warp >> 2) * (kOzWBN / 2);
    const uint32_t te = oz_u32(tempty) & kPeerMask;
    int it = 0;
    for (int tt = pfirst; tt < ntiles; tt += pstep) {
      int m0, n0;
      tile_origin(tt, m0, n0);
      const int row = m0 + q * 32 + lane;
      const bool rok = row < p.M;
      const int er = rok ? p.ea[row] : 0;
      const int lp = __ffs(p.panel) - 1;
      double* crow = p.C + (size_t)row * p.panel;
      const size_t sstride = (size_t)p.M * p.panel;
      for (int pass = 1; pass >= 0; --pass, ++it) {
        oz_mbar_wait(tfull, it & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int dmin = pass ? NS / 2 : 0;
        // 32 columns at a time (all 64 in registers at once spilled: 663 vs 633 ms per C5 call; an L1
        // prefetch of pass 0's read-modify-write lines: 647 ms)
#pragma unroll 1
        for (int half = 0; half < 2; ++half) {
          const int ch = ch0 + half * 32;
          double acc[32];
#pragma unroll
          for (int c = 0; c < 32; ++c) acc[c] = 0.0;
#pragma unroll
          for (int dl = NS / 2 - 1; dl >= 0; --dl) {  // smallest terms first
            const double sc = ldexp(1.0, -7 * (dmin + dl + 2));
            uint32_t v[32];
            const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(dl * kOzWBN + ch);
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                  "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                  "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int c = 0; c < 32; ++c) acc[c] = fma((double)(int)v[c], sc, acc[c]);
          }
          if (half == 1) {
            // every accumulator of this pass is in registers / stored: hand TMEM back to the MMA issuer
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(te) : "memory");
          }
          if (rok) {
            // 32-byte stores (one full sector per lane and instruction; the lanes of a warp are 64 /
            // 128 bytes apart in the panel layout, so 16-byte stores cost two half-filled sector
            // writes each)
#pragma unroll
            for (int c = 0; c < 32; c += 4) {
              const int col = n0 + ch + c;
              FFS_CHECK(col + 3 < p.N);
              const int4 e4 = *reinterpret_cast<const int4*>(p.eb + col);
              const int eb4[4] = {e4.x, e4.y, e4.z, e4.w};
              double o[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int bb = 1023 + er + eb4[u];  // 2^(ea + eb) from its biased exponent
                const double sf = (bb > 0 && bb < 2047) ? __longlong_as_double((long long)bb << 52) : ldexp(1.0, er + eb4[u]);
                o[u] = acc[c + u] * sf;
              }
              double* dst = crow + (size_t)(col >> lp) * sstride + (col & (p.panel - 1));
              if (pass == 0) {  // add the large terms to pass 1's sum of the small ones
                double pv[4];
                asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(pv[0]), "=d"(pv[1]), "=d"(pv[2]), "=d"(pv[3]) : "l"(dst));
#pragma unroll
                for (int u = 0; u < 4; ++u) o[u] += pv[u];
              }
              asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(dst), "d"(o[0]), "d"(o[1]), "d"(o[2]), "d"(o[3]) : "memory");
            }
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  oz2_cluster_sync();  // neither CTA leaves while the other may still signal it or read its TMEM
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
}

// x = 2^e sum_i q_i 2^{-7(i+1)}, |q_i| <= 127 (frexp exponent: |x 2^-e| < 1); q_i of element k of
// row r goes to out[(i * rows + r) * Kp + k]; zero for k in [K, Kp)
template <int NS>
__device__ __forceinline__ void oz_split_value(double v, int ex, int8_t (&q)[NS]) {
  double r = ldexp(v, -ex);
#pragma unroll
  for (int i = 0; i < NS; ++i) {
    const double f = trunc(r * 128.0);
    q[i] = (int8_t)f;
    r = r * 128.0 - f;
  }
}

// rows of a row-major [rows][ldx] fp64 matrix (one warp per row)
template <int NS>
static __global__ void ffs_ozaki_split_rows_kernel(const double* __restrict__ X, int rows, int K, int64_t ldx,
                                                   int8_t* __restrict__ out, int Kp, int* __restrict__ e) {
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= rows) return;
  const double* xr = X + (size_t)r * ldx;
  double mx = 0.0;
  for (int k = lane; k < K; k += 32) mx = fmax(mx, fabs(xr[k]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  int ex = 0;
  if (mx > 0.0) frexp(mx, &ex);
  if (lane == 0) e[r] = ex;
  for (int k = lane; k < Kp; k += 32) {
    int8_t q[NS];
    oz_split_value<NS>(k < K ? xr[k] : 0.0, ex, q);
#pragma unroll
    for (int i = 0; i < NS; ++i) out[((size_t)i * rows + r) * Kp + k] = q[i];
  }
}

// columns of a row-major [K][ldy] fp64 matrix (32 columns per CTA of 256 threads): column c's
// slices are written K-major, out[(i * ncols + c) * Kp + k]
template <int NS>
static __global__ void __launch_bounds__(256) ffs_ozaki_split_cols_kernel(const double* __restrict__ Y, int K, int ncols,
                                                                         int64_t ldy, int8_t* __restrict__ out, int Kp,
                                                                         int* __restrict__ e) {
  __shared__ double tile[64][33];
  __shared__ double red[8][32];
  const int c0 = blockIdx.x * 32, t = threadIdx.x, cl = t & 31, kg = t >> 5;
  double mx = 0.0;
  for (int k = kg; k < K; k += 8) mx = fmax(mx, fabs(Y[(size_t)k * ldy + c0 + cl]));
  red[kg][cl] = mx;
  __syncthreads();
  if (kg == 0) {
    for (int q = 1; q < 8; ++q) mx = fmax(mx, red[q][cl]);
    int ex = 0;
    if (mx > 0.0) frexp(mx, &ex);
    red[0][cl] = (double)ex;
    if (c0 + cl < ncols) e[c0 + cl] = ex;
  }
  __syncthreads();
  for (int kb = 0; kb < Kp; kb += 64) {
    for (int q = t; q < 64 * 32; q += 256) {
      const int kk = q >> 5, cc = q & 31;
      tile[kk][cc] = (kb + kk < K) ? Y[(size_t)(kb + kk) * ldy + c0 + cc] : 0.0;
    }
    __syncthreads();
    {
      const int cc = t >> 3, k8 = (t & 7) * 8;  // 32 columns x 8 groups of 8 k
      const int ex = (int)red[0][cc];
      int8_t q8[NS][8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        int8_t q[NS];
        oz_split_value<NS>(tile[k8 + u][cc], ex, q);
#pragma unroll
        for (int i = 0; i < NS; ++i) q8[i][u] = q[i];
      }
#pragma unroll
      for (int i = 0; i < NS; ++i) {
        uint64_t w = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) w |= (uint64_t)(uint8_t)q8[i][u] << (8 * u);
        *reinterpret_cast<uint64_t*>(out + ((size_t)i * ncols + c0 + cc) * Kp + kb + k8) = w;
      }
    }
    __syncthreads();
  }
}

}  // namespace ffsk
