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
template <int kGK, int kGStages>
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
};

template <typename T, int B, int kGjTJ>
__host__ __device__ inline size_t dense_gj_smem(int k0) {
  return sizeof(T) * ((size_t)B * k0 + 4 * B * kGjTJ + B * kGjTJ + B * B + B) + sizeof(int) * 2 * B;
}

// CPT adjacent columns per thread (2 for real: 16-byte W accesses), kGjTJ = 64 * CPT columns per
// CTA of 256 threads; the i loops keep UNR independent W loads in flight per thread.
template <typename T, int B, int kGjTJ>
static __global__ void __launch_bounds__(256) ffs_dense_gj_kernel(const DenseGjParams q) {
  using S = Sc<T>;
  constexpr int CPT = kGjTJ / 64;
  constexpr int UNR = 8;
  static_assert(CPT == 1 || (CPT == 2 && sizeof(T) == 8), "two columns per thread only for real");
  extern __shared__ __align__(16) unsigned char smem[];
  const int k0 = q.k0, k1 = k0 + B, Np = q.Np, N = q.N;
  const int sl = blockIdx.y;
  const int64_t i_s = q.base + sl;
  const int t = threadIdx.x, jg = t % 64, part = t / 64;
  const int jl = jg * CPT;                        // first column of this thread within the tile
  const int j = k1 + blockIdx.x * kGjTJ + jl;     // first global column
  const bool has = j < Np;
  const bool full = j + CPT - 1 < Np;             // every column of the group in range
  T* Vn = reinterpret_cast<T*>(smem);   // [B][k0]   V[X_new, 0:k0]
  T* Zp = Vn + (size_t)B * k0;          // [4][B][TJ] partial sums (negated)
  T* Zs = Zp + 4 * B * kGjTJ;           // [B][TJ]
  T* RP = Zs + B * kGjTJ;               // Row [B][B], Pinv [B]
  int* xn = reinterpret_cast<int*>(RP + B * B + B);
  const int32_t* pm = q.perm + i_s * Np;
  const T* Ug = reinterpret_cast<const T*>(q.U);
  T* W = reinterpret_cast<T*>(q.W) + (size_t)sl * Np * Np;
  if (t < B) xn[t] = q.positions[i_s * Np + k0 + t];
  if (t < B * B + B) RP[t] = reinterpret_cast<const T*>(q.rowg)[(size_t)sl * (B * B + B) + t];
  __syncthreads();
  for (int idx = t; idx < B * k0; idx += blockDim.x) {
    const int tt = idx / k0, ii = idx % k0;
    Vn[idx] = Ug[(size_t)xn[tt] * N + pm[ii]];
  }
  __syncthreads();
  auto ldw = [&](int ii, T (&w)[CPT]) {
    const T* src = W + (size_t)ii * Np + j;
    if constexpr (CPT == 2) {
      if (full) {
        const double2 v = *reinterpret_cast<const double2*>(src);
        w[0] = v.x;
        w[1] = v.y;
      } else {
        w[0] = src[0];
        w[1] = S::zero();
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
    for (; ii + 4 * (UNR - 1) < k0; ii += 4 * UNR) {
      T w[UNR][CPT];
#pragma unroll
      for (int u = 0; u < UNR; ++u) ldw(ii + 4 * u, w[u]);
#pragma unroll
      for (int u = 0; u < UNR; ++u)
#pragma unroll
        for (int tt = 0; tt < B; ++tt) {
          const T vn = Vn[tt * k0 + ii + 4 * u];
#pragma unroll
          for (int e = 0; e < CPT; ++e) acc[e][tt] = S::fms(vn, w[u][e], acc[e][tt]);
        }
    }
    for (; ii < k0; ii += 4) {
      T w[CPT];
      ldw(ii, w);
#pragma unroll
      for (int tt = 0; tt < B; ++tt)
#pragma unroll
        for (int e = 0; e < CPT; ++e) acc[e][tt] = S::fms(Vn[tt * k0 + ii], w[e], acc[e][tt]);
    }
  }
#pragma unroll
  for (int e = 0; e < CPT; ++e)
#pragma unroll
    for (int tt = 0; tt < B; ++tt) Zp[(part * B + tt) * kGjTJ + jl + e] = acc[e][tt];
  __syncthreads();
  // (2) one thread per column: Z = S^{-1} (V[X_new, j] - sum)
  if (t < kGjTJ && k1 + blockIdx.x * kGjTJ + t < Np) {
    const int c = t, jc = k1 + blockIdx.x * kGjTJ + c;
    T z[B];
#pragma unroll
    for (int tt = 0; tt < B; ++tt) {
      const T a01 = S::add(Zp[(0 * B + tt) * kGjTJ + c], Zp[(1 * B + tt) * kGjTJ + c]);
      const T a23 = S::add(Zp[(2 * B + tt) * kGjTJ + c], Zp[(3 * B + tt) * kGjTJ + c]);
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
      const T* wb = W + (size_t)ii * Np + k0;  // the same B scalars for every thread: L1 broadcast
#pragma unroll
      for (int tt = 0; tt < B; ++tt) {
        const T wv = wb[tt];
#pragma unroll
        for (int e = 0; e < CPT; ++e) a[e] = S::fms(wv, z[e][tt], a[e]);
      }
      T* dst = W + (size_t)ii * Np + j;
      if constexpr (CPT == 2) {
        if (full) *reinterpret_cast<double2*>(dst) = make_double2(a[0], a[1]);
        else dst[0] = a[0];
      } else {
        dst[0] = a[0];
      }
    };
    int ii = part;
    for (; ii + 4 * (UNR - 1) < k0; ii += 4 * UNR) {
      T a[UNR][CPT];
#pragma unroll
      for (int u = 0; u < UNR; ++u) ldw(ii + 4 * u, a[u]);
#pragma unroll
      for (int u = 0; u < UNR; ++u) upd(ii + 4 * u, a[u]);
    }
    for (; ii < k0; ii += 4) {
      T a[CPT];
      ldw(ii, a);
      upd(ii, a);
    }
  }
  // next block's Y_s columns (the tile holding columns k1 .. k1+B-1)
  if (blockIdx.x == 0 && q.Y != nullptr) {  // (no Y when every block is contracted gathered)
    __syncthreads();
    const int nb1 = min(B, Np - k1);
    const int64_t col0 = (int64_t)sl * B;
    for (int idx = t; idx < k1 * B; idx += blockDim.x) {
      const int ii = idx / B, c = idx % B;
      dense_y_store<T>(q.Y, q.ldY, pm[ii], col0 + c, c < nb1 ? S::neg(W[(size_t)ii * Np + k1 + c]) : S::zero());
    }
    if (t < nb1) dense_y_store<T>(q.Y, q.ldY, pm[k1 + t], col0 + t, S::one());
  }
}

}  // namespace ffsk
