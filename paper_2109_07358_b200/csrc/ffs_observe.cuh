// Observables of the samples, on the device: occupation numbers, pair
// occupations in a site window, and the Slater-Jastrow / Gutzwiller reweighting of Supp S5
// (PAPER.md:336-350): <O> = <J^2 o>_0 / <J^2>_0 with J = exp(-V/2 sum_i n_{i,up} n_{i,down})
// (Eq. 4), so J^2 = exp(-V D), D = number of doubly occupied sites. A spinful sample
// is the pair of rows (2s, 2s+1) = (up, down) of an FFS positions array.
//
// All three are HBM-bound reductions over the int32 positions [M][N'] (4 N' bytes per sample):
// positions are read once, coalesced; counts go to shared-memory histograms where they fit and
// are flushed with one 64-bit atomic per nonzero bin. The reweighted averages are formed from
// integer histograms by D (exact, order-independent): sum_s J_s^2 O_s = sum_D exp(-V D) H_O(D).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ffsk {

constexpr int kObsThreads = 256;

// occ[x] += number of samples with x occupied; entries < 0 (L-ensemble padding) skipped.
// SMEM: per-CTA u32 histogram of L bins (L <= 49152), else direct global atomics.
template <bool SMEM>
static __global__ void __launch_bounds__(kObsThreads) ffs_occupation_kernel(const int32_t* __restrict__ pos,
                                                                           int64_t n, int L,
                                                                           unsigned long long* __restrict__ occ) {
  extern __shared__ unsigned int hist[];
  if constexpr (SMEM) {
    for (int x = threadIdx.x; x < L; x += blockDim.x) hist[x] = 0;
    __syncthreads();
  }
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
  for (int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; q < n; q += stride) {
    int v[4];
    if (q + 3 < n && ((reinterpret_cast<uintptr_t>(pos + q) & 15) == 0)) {
      const int4 w = __ldg(reinterpret_cast<const int4*>(pos + q));
      v[0] = w.x; v[1] = w.y; v[2] = w.z; v[3] = w.w;
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = q + u < n ? pos[q + u] : -1;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (v[u] < 0 || v[u] >= L) continue;
      if constexpr (SMEM) atomicAdd(&hist[v[u]], 1u);
      else atomicAdd(&occ[v[u]], 1ull);
    }
  }
  if constexpr (SMEM) {
    __syncthreads();
    for (int x = threadIdx.x; x < L; x += blockDim.x)
      if (hist[x]) atomicAdd(&occ[x], (unsigned long long)hist[x]);
  }
}

// pair[x][y] += number of samples with x and y occupied (x, y < W); one warp per sample, its
// in-window sites gathered to shared memory first
static __global__ void __launch_bounds__(kObsThreads) ffs_pair_kernel(const int32_t* __restrict__ pos, int64_t M,
                                                                     int Np, int W,
                                                                     unsigned long long* __restrict__ pair) {
  extern __shared__ int sites[];  // [warps][Np]
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int* my = sites + wid * Np;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + wid; i < M; i += nw) {
    int cnt = 0;
    for (int k0 = 0; k0 < Np; k0 += 32) {
      const int k = k0 + lane;
      const int x = k < Np ? pos[i * Np + k] : -1;
      const bool in = x >= 0 && x < W;
      const unsigned b = __ballot_sync(0xffffffffu, in);
      if (in) my[cnt + __popc(b & ((1u << lane) - 1u))] = x;
      cnt += __popc(b);
    }
    __syncwarp();
    for (int q = lane; q < cnt * cnt; q += 32) {
      const int a = q / cnt, c = q - a * cnt;
      atomicAdd(&pair[(int64_t)my[a] * W + my[c]], 1ull);
    }
    __syncwarp();
  }
}

// Gutzwiller histograms of Ms spinful samples: dcount[D] += 1 and occ_d[D][x] += n_x(up) + n_x(dn)
// per sample with D doubly occupied sites. One warp per spinful sample; the up row is marked in a
// per-warp bitmap of L bits in shared memory, the down row counts the marked sites.
static __global__ void __launch_bounds__(kObsThreads) ffs_gutzwiller_kernel(const int32_t* __restrict__ pos,
                                                                           int64_t Ms, int Np, int L,
                                                                           unsigned long long* __restrict__ dcount,
                                                                           unsigned long long* __restrict__ occ_d) {
  extern __shared__ unsigned int bits[];  // [warps][ceil(L/32)]
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int words = (L + 31) >> 5;
  unsigned int* my = bits + (size_t)wid * words;
  for (int q = lane; q < words; q += 32) my[q] = 0u;
  __syncwarp();
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t s = (int64_t)blockIdx.x * (blockDim.x >> 5) + wid; s < Ms; s += nw) {
    const int32_t* up = pos + (2 * s) * Np;
    const int32_t* dn = up + Np;
    for (int k = lane; k < Np; k += 32) {
      const int x = up[k];
      if (x >= 0 && x < L) atomicOr(&my[x >> 5], 1u << (x & 31));
    }
    __syncwarp();
    int d = 0;
    for (int k = lane; k < Np; k += 32) {
      const int x = dn[k];
      if (x >= 0 && x < L && ((my[x >> 5] >> (x & 31)) & 1u)) ++d;
    }
    d = __reduce_add_sync(0xffffffffu, d);
    if (lane == 0) atomicAdd(&dcount[d], 1ull);
    unsigned long long* od = occ_d + (int64_t)d * L;
    for (int k = lane; k < 2 * Np; k += 32) {
      const int x = up[k];  // up row then down row (contiguous)
      if (x >= 0 && x < L) atomicAdd(&od[x], 1ull);
    }
    __syncwarp();
    for (int k = lane; k < Np; k += 32) {  // clear the bitmap for the next sample
      const int x = up[k];
      if (x >= 0 && x < L) my[x >> 5] = 0u;
    }
    __syncwarp();
  }
}

// result[0] = <J^2>_0 = sum_D w_D c_D / Ms, result[1] = <D>_J, result[2 + x] = <n_x>_J with
// w_D = exp(-V D); sums over D in ascending order (one thread per output)
static __global__ void ffs_reweight_finalize_kernel(const unsigned long long* __restrict__ dcount,
                                                    const unsigned long long* __restrict__ occ_d, int Dmax, int L,
                                                    int64_t Ms, double V, double* __restrict__ result) {
  double Z = 0.0, Dn = 0.0;
  for (int d = 0; d <= Dmax; ++d) {
    const double w = exp(-V * (double)d) * (double)dcount[d];
    Z += w;
    Dn += w * (double)d;
  }
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t == 0) {
    result[0] = Z / (double)Ms;
    result[1] = Dn / Z;
  }
  for (int64_t x = t; x < L; x += (int64_t)gridDim.x * blockDim.x) {
    double num = 0.0;
    for (int d = 0; d <= Dmax; ++d) num += exp(-V * (double)d) * (double)occ_d[(int64_t)d * L + x];
    result[2 + x] = num / Z;
  }
}

}  // namespace ffsk
