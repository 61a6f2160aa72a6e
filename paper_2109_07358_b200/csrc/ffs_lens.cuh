// L-ensemble DPP front end (text-summarisation pipeline, step 2): with the
// correlation matrix C = sum_j lambda_j v_j v_j^T, "each eigenvector u_j is selected with
// probability lambda_j/(lambda_j+1)" and the selected vectors form the U of Eq. 1 that FFS samples
// with its own particle number N_i. This kernel draws, per sample, the kept set (ascending j) from
// the keep uniforms, applies the FFS permutation of the N_i kept columns (reading Q6 with N = N_i)
// to it, and writes the sample's column list and N_i; ffs_sample_kernel then runs N_i steps on
// those columns of V (ragged mode).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ffsk {

// one thread per sample; kept list in shared memory, interleaved across the block ([K][blockDim])
// so the threads of a warp touch consecutive words
static __global__ void ffs_lens_prep_kernel(const double* __restrict__ lambda, const double* __restrict__ uniforms,
                                            int32_t* __restrict__ cols, int32_t* __restrict__ nps, int64_t M, int K) {
  extern __shared__ int lscratch[];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int* a = lscratch + threadIdx.x;
  const int bs = blockDim.x;
  if (i >= M) return;
  const double* u = uniforms + i * 3 * (int64_t)K;
  int n = 0;
  for (int j = 0; j < K; ++j) {
    const double lj = lambda[j];
    if (u[j] < lj / (lj + 1.0)) a[(n++) * bs] = j;  // fp64 keep decision, as the oracle takes it
  }
  // forward partial Fisher-Yates over the n kept columns; the swaps act on the kept list itself,
  // so a[j] = kept[m_j] (the oracle permutes the columns of U_i = V[:, kept])
  for (int j = 0; j < n; ++j) {
    const int nn = n - j;
    int r = (int)floor(u[K + j] * (double)nn);
    r = (r > nn - 1 ? nn - 1 : r) + j;
    const int t = a[j * bs];
    a[j * bs] = a[r * bs];
    a[r * bs] = t;
    cols[i * K + j] = a[j * bs];
  }
  FFS_CHECK(n >= 0 && n <= K);
  nps[i] = n;
}

}  // namespace ffsk
