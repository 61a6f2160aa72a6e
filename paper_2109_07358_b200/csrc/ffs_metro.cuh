// Continuous / large-L variant of FFS (Supp S7): per step k the conditional
// P(x_k | x_<k; m) ∝ |u_x^T h|^2 is sampled by a Metropolis chain of M_cond updates instead of the
// explicit inverse-CDF draw over all L sites, so the cost per sample is O(N'^3 + M_cond N'^2),
// independent of L. Readings (Q16-Q18, shared with the oracle):
// start x = floor(u_init L); discrete update x' = floor(u_prop L) (uniform, symmetric proposal);
// accept iff u_acc w(x) < w(x'); chosen sites have weight 0.
//
// One warp per sample. The coefficients W = A^{-1} V[X, later columns] live in global memory per
// warp slot and get a rank-1 Gauss-Jordan update after every step (O(k N') per step, lanes over
// columns, coalesced rows). The chain's weights s(x) = V[x, 0:k+1] . (-W[0:k, k]; 1) of all
// M_cond + 1 states (start + proposals) are independent of the acceptance history: with h
// scattered into U's column order each is one coalesced read of row x by the warp and a warp
// reduction, 8 states' reads in flight together; one lane then runs the sequential accept/reject
// chain over the stored weights.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ffs_scalar.cuh"

namespace ffsk {

struct MetroParams {
  const double* U;         // [L][N] row-major scalars (complex interleaved)
  const int32_t* perm;     // [M][Np] permutation prefixes (ffs_permute_kernel)
  const double* uniforms;  // [M][Np + Np (1 + 2 Mc)]
  int32_t* positions;      // [M][Np]
  int32_t* flags;          // [M] or null: bit0 non-finite pivot, bit2 chain ended on a zero-weight site
  double* wbuf;            // per warp slot [Np][Np] scalars
  int64_t M;
  int L, N, Np, Mc;
};

constexpr int kMetroWarps = 8;

__device__ __forceinline__ double ldg_t(const double* p) { return __ldg(p); }
__device__ __forceinline__ cplx ldg_t(const cplx* p) {
  const double2 d = __ldg(reinterpret_cast<const double2*>(p));
  return {d.x, d.y};
}

__host__ __device__ inline size_t metro_align(size_t v) { return (v + 15) & ~size_t(15); }

// per-warp shared memory: m [Np] int, pos [Np] int, h [Np] T, vrow [Np] T, chain entries [Mc + 1]
// of (s T, w double, x int), pivot T, hp [N] T
template <typename T>
__host__ __device__ inline size_t metro_warp_smem(int Np, int Mc, int N) {
  const size_t e = (size_t)Mc + 1;
  return 2 * metro_align(sizeof(int) * Np) + 2 * metro_align(sizeof(T) * Np) +
         metro_align(e * (sizeof(int) + sizeof(double) + sizeof(T))) + metro_align(sizeof(T)) +
         metro_align(sizeof(T) * N);
}

template <typename T>
static __global__ void __launch_bounds__(kMetroWarps * 32) ffs_metro_kernel(const MetroParams p) {
  using S = Sc<T>;
  extern __shared__ __align__(16) unsigned char msm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int L = p.L, N = p.N, Np = p.Np, Mc = p.Mc;
  const int E = Mc + 1;
  unsigned char* b = msm + (size_t)wid * metro_warp_smem<T>(Np, Mc, N);
  int* perm = reinterpret_cast<int*>(b);
  b += metro_align(sizeof(int) * Np);
  int* pos = reinterpret_cast<int*>(b);
  b += metro_align(sizeof(int) * Np);
  T* h = reinterpret_cast<T*>(b);
  b += metro_align(sizeof(T) * Np);
  T* vrow = reinterpret_cast<T*>(b);
  b += metro_align(sizeof(T) * Np);
  T* es = reinterpret_cast<T*>(b);            // [E] s of each chain entry
  double* ew = reinterpret_cast<double*>(es + E);  // [E] weights
  int* ex = reinterpret_cast<int*>(ew + E);   // [E] sites
  b += metro_align((size_t)E * (sizeof(int) + sizeof(double) + sizeof(T)));
  T* pivot = reinterpret_cast<T*>(b);
  b += metro_align(sizeof(T));
  T* hp = reinterpret_cast<T*>(b);
  const T* Ug = reinterpret_cast<const T*>(p.U);
  const int64_t slot = (int64_t)blockIdx.x * kMetroWarps + wid;
  const int64_t nslots = (int64_t)gridDim.x * kMetroWarps;
  T* W = reinterpret_cast<T*>(p.wbuf) + slot * (int64_t)Np * Np;
  const int64_t ustride = (int64_t)Np + (int64_t)Np * (1 + 2 * Mc);

  for (int64_t i = slot; i < p.M; i += nslots) {
    const double* urow = p.uniforms + i * ustride;
    for (int j = lane; j < Np; j += 32) perm[j] = p.perm[i * Np + j];
    __syncwarp();
    int flag = 0;
    for (int k = 0; k < Np; ++k) {
      // h = (-W[0:k, k]; 1): s(x) = V[x, k] - V[x, 0:k] W[0:k, k] = V[x, 0:k+1] . h
      for (int j = lane; j < k; j += 32) h[j] = S::neg(W[(size_t)j * Np + k]);
      if (lane == 0) h[k] = S::one();
      __syncwarp();
      const double* uc = urow + Np + (int64_t)k * (1 + 2 * Mc);
      // h scattered into U's column order (hp[m_j] = h[j] for j <= k, 0 elsewhere): a chain state's
      // s(x) = U[x, :] . hp is then one coalesced read of row x by the warp and a warp reduction
      for (int c = lane; c < N; c += 32) hp[c] = S::zero();
      __syncwarp();
      for (int j = lane; j <= k; j += 32) hp[perm[j]] = h[j];
      __syncwarp();
      // weights of the start (e = 0) and the Mc proposals (e >= 1), kBatch states at a time (their
      // row reads in flight together)
      constexpr int kBatch = 8;
      for (int e0 = 0; e0 < E; e0 += kBatch) {
        int xb[kBatch];
        bool live[kBatch];
        T part[kBatch];
#pragma unroll
        for (int b = 0; b < kBatch; ++b) {
          const int e = e0 + b;
          int x = 0;
          bool chosen = true;
          if (e < E) {
            x = (int)floor(uc[e == 0 ? 0 : 2 * e - 1] * (double)L);
            x = x > L - 1 ? L - 1 : x;
            bool hit = false;
            for (int j = lane; j < k; j += 32) hit |= (pos[j] == x);
            chosen = __any_sync(0xffffffffu, hit);
          }
          xb[b] = x;
          live[b] = !chosen;
          part[b] = S::zero();
        }
        for (int c = lane; c < N; c += 32) {
          const T hc = hp[c];
#pragma unroll
          for (int b = 0; b < kBatch; ++b)
            if (live[b]) part[b] = S::fms(S::neg(ldg_t(Ug + (size_t)xb[b] * N + c)), hc, part[b]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int b = 0; b < kBatch; ++b) {
            if constexpr (sizeof(T) == 8) {
              part[b] = S::add(part[b], __shfl_xor_sync(0xffffffffu, part[b], o));
            } else {
              cplx y;
              y.re = __shfl_xor_sync(0xffffffffu, part[b].re, o);
              y.im = __shfl_xor_sync(0xffffffffu, part[b].im, o);
              part[b] = S::add(part[b], y);
            }
          }
        if (lane == 0) {
#pragma unroll
          for (int b = 0; b < kBatch; ++b)
            if (e0 + b < E) {
              ex[e0 + b] = xb[b];
              ew[e0 + b] = live[b] ? S::abs2(part[b]) : 0.0;
              es[e0 + b] = live[b] ? part[b] : S::zero();
            }
        }
      }
      __syncwarp();
      // the sequential accept / reject chain
      if (lane == 0) {
        int cur = 0;
        double wc = ew[0];
        for (int t = 1; t <= Mc; ++t) {
          const double ua = uc[2 * t];
          if (ua * wc < ew[t]) {
            cur = t;
            wc = ew[t];
          }
        }
        if (!(wc > 0.0)) flag |= 4;
        FFS_CHECK(ex[cur] >= 0 && ex[cur] < L);
        pos[k] = ex[cur];
        *pivot = es[cur];  // s(x_k): the new diagonal entry of the factorization
      }
      __syncwarp();
      if (k + 1 < Np) {
        const int xk = pos[k];
        // the new row V[x_k, :] in permuted column order
        for (int j = lane; j < Np; j += 32) vrow[j] = Ug[(size_t)xk * N + perm[j]];
        const T ip = S::recip(*pivot);
        if (!S::finite(ip)) flag |= 1;
        __syncwarp();
        // rank-1 Gauss-Jordan update (A bordered by row x_k, column k):
        // z_j = (V[x_k, j] - V[x_k, 0:k] W[0:k, j]) / s(x_k);  W[0:k, j] += h[0:k] z_j;  W[k, j] = z_j
        for (int j = k + 1 + lane; j < Np; j += 32) {
          T z = vrow[j];
          for (int ii = 0; ii < k; ++ii) z = S::fms(vrow[ii], W[(size_t)ii * Np + j], z);
          z = S::mul(z, ip);
          for (int ii = 0; ii < k; ++ii) W[(size_t)ii * Np + j] = S::fms(S::neg(h[ii]), z, W[(size_t)ii * Np + j]);
          W[(size_t)k * Np + j] = z;
        }
      }
      __syncwarp();
    }
    for (int j = lane; j < Np; j += 32) p.positions[i * Np + j] = pos[j];
    flag = __reduce_or_sync(0xffffffffu, flag);
    if (lane == 0 && p.flags) p.flags[i] = flag;
    __syncwarp();
  }
}

}  // namespace ffsk
