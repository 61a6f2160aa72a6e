// Latency of one FFS draw step pieces in isolation (single warp, dependent iterations).
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2109_07358_b200/csrc/ffs_warp_kernel.cuh"
using namespace ffsk;
__global__ void kdraw(double* out, long long* cyc, int iters) {
  const int lane = threadIdx.x & 31;
  double col[8];
  for (int r = 0; r < 8; ++r) col[r] = 0.01 * (lane * 8 + r + 1);
  double u = 0.37, acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    Draw d = seg_draw<8, 32>(col, u, 0);
    const int own = __ffs(d.ball) - 1;
    const int orow = __shfl_sync(0xffffffffu, d.rsel, own);
    acc += orow;
    col[it & 7] += 1e-9 * (orow + 1);  // dependency on the result
  }
  long long t1 = clock64();
  if (lane == 0) cyc[0] = (t1 - t0) / iters;
  out[lane] = acc;
}
__global__ void kextract(double* out, long long* cyc, int iters) {
  const int lane = threadIdx.x & 31;
  double P[8][4];
  for (int r = 0; r < 8; ++r) for (int c = 0; c < 4; ++c) P[r][c] = lane * 0.1 + r + c * 0.01;
  int own = 3, rs = lane & 7;
  double acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    double prow[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      double t[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) t[r] = P[r][c];
#pragma unroll
      for (int w = 1; w < 8; w <<= 1)
#pragma unroll
        for (int i = 0; i < 8; i += 2 * w) t[i] = (rs & w) ? t[i + w] : t[i];
      prow[c] = __shfl_sync(0xffffffffu, t[0], own);
    }
    const double ip = fast_rcp(prow[1]);
    double sp2 = prow[2] * ip;
#pragma unroll
    for (int r = 0; r < 8; ++r) P[r][2] = fma(-P[r][1], sp2, P[r][2]);
    acc += P[0][2];
    own = (own + (prow[0] > 1e300 ? 1 : 0)) & 31;
    rs = (rs + (P[3][2] > 1e300 ? 1 : 0)) & 7;
  }
  long long t1 = clock64();
  if (lane == 0) cyc[1] = (t1 - t0) / iters;
  out[lane] = acc;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 16);
  kdraw<<<1, 32>>>(o, c, 100); kextract<<<1, 32>>>(o, c, 100); cudaDeviceSynchronize();
  kdraw<<<1, 32>>>(o, c, 5000); kextract<<<1, 32>>>(o, c, 5000); cudaDeviceSynchronize();
  long long h[2]; cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
  printf("{\"draw_cycles\": %lld, \"extract_rcp_update_cycles\": %lld}\n", h[0], h[1]);
}
