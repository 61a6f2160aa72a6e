// GPU modified-HKPV sampler (the paper's comparison method): the chain rule
// on the projection kernel K = U U^dagger (steps as SPEC.md:238-246). With
// residuals r(x) = |u_x|^2 - sum_{j<k} |<u_x, e_j>|^2, step k draws x_k ∝ r (selection rule of
// reading Q5), orthonormalises u_{x_k} against e_1..e_{k-1} (classical Gram-Schmidt, two passes),
// and subtracts |<u_x, e_k>|^2 from every residual: 2 L N multiply-adds per step, 2 L N^2 per
// sample, against FFS's L N^2 + N^3.
//
// B200 form: the samples of a batch advance in lockstep, so the residual update of step k for
// all S batch samples is ONE dense GEMM C = U conj(E_k) (L x N x S, U shared by every sample) on
// the FP64 tensor pipe (ffs_dgemm_kernel<..., EPI = 1>, which subtracts |C|^2 from r in its
// epilogue instead of storing C); the draw and the Gram-Schmidt step are one CTA per sample
// (ffs_hkpv_step_kernel). The FFS path this is compared with is ffs_sample (same selection rule,
// same uniforms layout for the selections).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ffs_dense.cuh"
#include "ffs_kernel.cuh"

namespace ffsk {

struct HkpvParams {
  const double* U;         // [L][Kp] zero-padded copy of U (scalars of T)
  int64_t ldu;             // row stride of U in scalars of T
  const double* uniforms;  // [M][Np] selection draws
  int32_t* positions;      // [M][Np]
  int32_t* flags;          // [M] or null
  double* r;               // [S][L] residuals of the batch
  uint32_t* chosen;        // [S][(L + 31) / 32]
  double* E;               // [S][Np][N] scalars of T: e_1 .. e_{N'-1}
  double* Eb;              // GEMM operand: conj(e_k) of every batch sample, [fK][ldE] (complex: real expansion)
  int64_t ldE;             // columns of Eb in scalars of T
  int64_t base;            // first sample of the batch
  int L, N, Np, k, Sb;
};

constexpr int kHkpvThreads = 256;

__device__ __forceinline__ double conj_t(double a) { return a; }
__device__ __forceinline__ cplx conj_t(cplx a) { return {a.re, -a.im}; }

// r[s][x] = |u_x|^2 for the Sb batch samples; chosen bitmaps cleared
template <typename T>
static __global__ void ffs_hkpv_init_kernel(const HkpvParams p) {
  using S = Sc<T>;
  const T* U = reinterpret_cast<const T*>(p.U);
  const int words = (p.L + 31) / 32;
  const int64_t n = (int64_t)p.Sb * p.L;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(q % p.L);
    double a = 0.0;
    for (int c = 0; c < p.N; ++c) a += S::abs2(U[(size_t)x * p.ldu + c]);
    p.r[q] = a;
  }
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < (int64_t)p.Sb * words;
       q += (int64_t)gridDim.x * blockDim.x)
    p.chosen[q] = 0u;
}

__device__ __forceinline__ double hk_block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
  return s;
}

// step k of one batch sample (CTA): draw x_k from the residuals, then (k < N'-1) e_k by two
// classical Gram-Schmidt passes against e_0 .. e_{k-1}, written to E and to the GEMM operand
template <typename T>
static __global__ void __launch_bounds__(kHkpvThreads) ffs_hkpv_step_kernel(const HkpvParams p) {
  using S = Sc<T>;
  extern __shared__ __align__(16) unsigned char hsm[];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nwarp = blockDim.x >> 5;
  const int sl = blockIdx.x;
  const int64_t i = p.base + sl;
  const int L = p.L, N = p.N, Np = p.Np, k = p.k;
  double* red = reinterpret_cast<double*>(hsm);              // [32]
  int* redi = reinterpret_cast<int*>(red + 32);              // [96]
  T* us = reinterpret_cast<T*>(redi + 96);                   // [N] the new row / its residual vector
  T* cf = us + N;                                            // [Np] Gram-Schmidt coefficients
  double* r = p.r + (size_t)sl * L;
  uint32_t* ch = p.chosen + (size_t)sl * ((L + 31) / 32);
  auto wgt = [&](int x) {
    const double v = r[x];
    return (((ch[x >> 5] >> (x & 31)) & 1u) || !(v > 0.0)) ? 0.0 : v;
  };
  // ---- draw: thread t owns the contiguous sites [t R, t R + R) (index order = scan order)
  const int R = (L + blockDim.x - 1) / blockDim.x;
  const int x0 = t * R, x1 = min(L, x0 + R);
  double loc = 0.0;
  for (int x = x0; x < x1; ++x) loc += wgt(x);
  double incl = loc;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += y;
  }
  __syncthreads();
  if (lane == 31) red[warp] = incl;
  __syncthreads();
  double woff = 0.0, Ttot = 0.0;
  for (int w = 0; w < nwarp; ++w) {
    if (w < warp) woff += red[w];
    Ttot += red[w];
  }
  const double excl = incl - loc + woff;
  const bool ok = Ttot > 0.0 && isfinite(Ttot);
  const double thr = p.uniforms[i * Np + k] * Ttot;
  constexpr int kNone = 0x7fffffff;
  int cf_first = kNone, cl_last = -1, cu_free = kNone;
  {
    double c = excl;
    for (int x = x0; x < x1; ++x) {
      const double w = wgt(x);
      c += w;
      if (w > 0.0) {
        if (cf_first == kNone && c > thr) cf_first = x;
        cl_last = x;
      }
      if (cu_free == kNone && !((ch[x >> 5] >> (x & 31)) & 1u)) cu_free = x;
    }
  }
  cf_first = __reduce_min_sync(0xffffffffu, cf_first);
  cl_last = __reduce_max_sync(0xffffffffu, cl_last);
  cu_free = __reduce_min_sync(0xffffffffu, cu_free);
  if (lane == 0) {
    redi[warp] = cf_first;
    redi[32 + warp] = cl_last;
    redi[64 + warp] = cu_free;
  }
  __syncthreads();
  int xs;
  {
    int a = kNone, b = -1, c = kNone;
    for (int w = 0; w < nwarp; ++w) {
      a = min(a, redi[w]);
      b = max(b, redi[32 + w]);
      c = min(c, redi[64 + w]);
    }
    xs = !ok ? c : (a != kNone ? a : b);
  }
  FFS_CHECK(xs >= 0 && xs < L);
  if (xs < 0 || xs >= L) xs = 0;  // unreachable for N' <= N <= L
  const double wsel = wgt(xs);
  __syncthreads();  // every thread has read the residuals / bitmap before the update below
  if (t == 0) {
    p.positions[i * Np + k] = xs;
    ch[xs >> 5] |= 1u << (xs & 31);
    if (p.flags) {
      const int f = (!ok ? 1 : 0) | ((ok && wsel / Ttot < 1e-12) ? 2 : 0);
      p.flags[i] = (k == 0 ? 0 : p.flags[i]) | f;
    }
  }
  if (k + 1 >= Np) return;
  // ---- e_k: u_{x_k} orthonormalised against e_0 .. e_{k-1} (two classical Gram-Schmidt passes)
  const T* U = reinterpret_cast<const T*>(p.U);
  const T* E = reinterpret_cast<const T*>(p.E) + (size_t)sl * Np * N;
  for (int n = t; n < N; n += blockDim.x) us[n] = U[(size_t)xs * p.ldu + n];
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass) {
    for (int j = warp; j < k; j += nwarp) {  // <v, e_j> = sum_n v_n conj(e_j,n), one warp per j
      T a = S::zero();
      for (int n = lane; n < N; n += 32) a = S::fms(S::neg(us[n]), conj_t(E[(size_t)j * N + n]), a);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        if constexpr (sizeof(T) == 8) {
          a = S::add(a, __shfl_xor_sync(0xffffffffu, a, o));
        } else {
          cplx b;
          b.re = __shfl_xor_sync(0xffffffffu, a.re, o);
          b.im = __shfl_xor_sync(0xffffffffu, a.im, o);
          a = S::add(a, b);
        }
      }
      if (lane == 0) cf[j] = a;
    }
    __syncthreads();
    for (int n = t; n < N; n += blockDim.x) {
      T v = us[n];
      for (int j = 0; j < k; ++j) v = S::fms(cf[j], E[(size_t)j * N + n], v);
      us[n] = v;
    }
    __syncthreads();
  }
  double nl = 0.0;
  for (int n = t; n < N; n += blockDim.x) nl += S::abs2(us[n]);
  const double nrm2 = hk_block_sum(nl, red);
  const double inv = 1.0 / sqrt(nrm2);
  T* Ek = reinterpret_cast<T*>(p.E) + ((size_t)sl * Np + k) * N;
  for (int n = t; n < N; n += blockDim.x) {
    const T e = S::mul(us[n], S::one()) ;
    T es;
    if constexpr (sizeof(T) == 8) es = e * inv;
    else es = {e.re * inv, e.im * inv};
    Ek[n] = es;
    dense_y_store<T>(p.Eb, p.ldE, n, (int64_t)sl, conj_t(es));
  }
}

// Small L (real, L <= 32 R): one warp per sample for all N' steps, U^T once per CTA in shared
// memory (the swizzled layout of ffs_sample_kernel's warp owners), the sample's residuals in
// registers (lane l owns sites l R .. l R + R - 1), its e-vectors in its shared-memory slice.
// Per step: the draw (select_site), Gram-Schmidt with lanes over the e-vectors / components, and
// the residual update r_x -= |u_x . e_k|^2 (R x N FMAs per lane from the shared U^T).
struct HkpvWarpParams {
  const double* U;         // [L][N]
  const double* uniforms;  // [M][Np]
  int32_t* positions;      // [M][Np]
  int32_t* flags;
  int64_t M;
  int L, N, Np, Lp, ut_stride;
  size_t ushared, owner_bytes;
};

// e-vector rows are N + 1 doubles apart: lanes over j reading E[j][n] hit distinct banks
__host__ __device__ inline size_t hkpv_warp_owner_bytes(int N, int Np) {
  return align16(sizeof(double) * (size_t)Np * (N + 1)) + align16(sizeof(double) * 2 * (size_t)N) +
         align16(sizeof(double) * (size_t)Np) + align16(sizeof(double) * 32 + sizeof(int) * 96);
}

template <int R, int MAXT>
static __global__ void __launch_bounds__(MAXT, 1) ffs_hkpv_warp_kernel(const HkpvWarpParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int L = p.L, N = p.N, Np = p.Np;
  double* Uts = reinterpret_cast<double*>(smem);
  for (int idx = threadIdx.x; idx < N * p.Lp; idx += blockDim.x) {
    const int x = idx / N, c = idx % N;
    Uts[(size_t)c * p.ut_stride + Swz<double, R>::phys(x)] = (x < L) ? p.U[(size_t)x * N + c] : 0.0;
  }
  __syncthreads();
  unsigned char* ob = smem + p.ushared + (size_t)wid * p.owner_bytes;
  const int ldE = N + 1;
  double* E = reinterpret_cast<double*>(ob);                                           // [Np][N + 1]
  double* v = reinterpret_cast<double*>(ob + align16(sizeof(double) * (size_t)Np * ldE));  // [N] (+ [N] scratch)
  double* cf = v + 2 * N;                                                          // [Np]
  double* red = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(cf) + align16(sizeof(double) * Np));
  int* redi = reinterpret_cast<int*>(red + 32);
  Params lp{};  // load_col needs only the shared-U^T stride
  lp.ut_stride = p.ut_stride;
  for (int64_t i = (int64_t)blockIdx.x * nwarps + wid; i < p.M; i += (int64_t)gridDim.x * nwarps) {
    double res[R];
    for (int r = 0; r < R; ++r) res[r] = 0.0;
    for (int c = 0; c < N; ++c) {
      double u[R];
      load_col<double, R, true>(lp, Uts, c, lane, u);
#pragma unroll
      for (int r = 0; r < R; ++r) res[r] = fma(u[r], u[r], res[r]);
    }
    uint32_t chosen = 0;
    int flag = 0;
    for (int k = 0; k < Np; ++k) {
      double w[R];
#pragma unroll
      for (int r = 0; r < R; ++r) w[r] = (((chosen >> r) & 1u) || !(res[r] > 0.0)) ? 0.0 : res[r];
      double T;
      const int xs = select_site<true, R>(w, p.uniforms[i * Np + k], lane, L, chosen, red, redi, T);
      if (!(T > 0.0 && isfinite(T))) flag |= 1;
      const int own = xs / R, orow = xs % R;
      if (lane == own) {
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (r == orow) {
            if (T > 0.0 && w[r] / T < 1e-12) flag |= 2;
            chosen |= 1u << r;
          }
        p.positions[i * Np + k] = xs;
      }
      FFS_CHECK(xs >= 0 && xs < L);
      if (k + 1 == Np) break;
      // e_k: two classical Gram-Schmidt passes of u_{x_k} against e_0 .. e_{k-1}
      for (int n = lane; n < N; n += 32) v[n] = Uts[(size_t)n * p.ut_stride + Swz<double, R>::phys(xs)];
      __syncwarp();
      for (int pass = 0; pass < 2; ++pass) {
        for (int j = lane; j < k; j += 32) {
          double a = 0.0;
          for (int n = 0; n < N; ++n) a = fma(v[n], E[(size_t)j * ldE + n], a);
          cf[j] = a;
        }
        __syncwarp();
        for (int n = lane; n < N; n += 32) {
          double a = v[n];
          for (int j = 0; j < k; ++j) a = fma(-cf[j], E[(size_t)j * ldE + n], a);
          v[n] = a;
        }
        __syncwarp();
      }
      double nl = 0.0;
      for (int n = lane; n < N; n += 32) nl = fma(v[n], v[n], nl);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) nl += __shfl_xor_sync(0xffffffffu, nl, o);
      const double inv = 1.0 / sqrt(nl);
      for (int n = lane; n < N; n += 32) E[(size_t)k * ldE + n] = v[n] * inv;
      __syncwarp();
      // r_x -= |u_x . e_k|^2 for this lane's sites
      double c[R];
#pragma unroll
      for (int r = 0; r < R; ++r) c[r] = 0.0;
      const double* ek = E + (size_t)k * ldE;
      for (int n = 0; n < N; ++n) {
        double u[R];
        load_col<double, R, true>(lp, Uts, n, lane, u);
        const double e = ek[n];
#pragma unroll
        for (int r = 0; r < R; ++r) c[r] = fma(u[r], e, c[r]);
      }
#pragma unroll
      for (int r = 0; r < R; ++r) res[r] = fma(-c[r], c[r], res[r]);
    }
    flag = __reduce_or_sync(0xffffffffu, flag);
    if (lane == 0 && p.flags) p.flags[i] = flag;
    __syncwarp();
  }
}

}  // namespace ffsk
