#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int iters) {
  __shared__ __align__(16) double dump[64];
  const int lane = threadIdx.x & 31;
  double P[8][4];
  for (int r = 0; r < 8; ++r) for (int c = 0; c < 4; ++c) P[r][c] = lane * 0.1 + r + c * 0.01;
  int own = 3, orow = 5;
  double acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (lane == own) {
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 4; c += 2) *reinterpret_cast<double2*>(dump + r * 4 + c) = make_double2(P[r][c], P[r][c + 1]);
    }
    __syncwarp();
    double2 a = *reinterpret_cast<double2*>(dump + orow * 4);
    double2 b = *reinterpret_cast<double2*>(dump + orow * 4 + 2);
    acc += a.x + b.y;
    own = ((int)(a.y * 7.0) + it) & 31;
    orow = ((int)(b.x * 3.0) + it) & 7;
    P[it & 7][it & 3] += 1e-3;
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) cyc[0] = (t1 - t0) / iters;
  out[lane] = acc;
}
__global__ void k2(double* out, long long* cyc, int iters) {  // shuffle-select variant
  const int lane = threadIdx.x & 31;
  double P[8][4];
  for (int r = 0; r < 8; ++r) for (int c = 0; c < 4; ++c) P[r][c] = lane * 0.1 + r + c * 0.01;
  int own = 3, rsel = lane & 7;
  double acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    double v[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      double a0 = (rsel & 1) ? P[1][c] : P[0][c], a1 = (rsel & 1) ? P[3][c] : P[2][c];
      double a2 = (rsel & 1) ? P[5][c] : P[4][c], a3 = (rsel & 1) ? P[7][c] : P[6][c];
      double b0 = (rsel & 2) ? a1 : a0, b1 = (rsel & 2) ? a3 : a2;
      v[c] = __shfl_sync(0xffffffffu, (rsel & 4) ? b1 : b0, own);
    }
    acc += v[0] + v[3];
    own = ((int)(v[1] * 7.0) + it) & 31;
    rsel = ((int)(v[2] * 3.0) + it + lane) & 7;
    P[it & 7][it & 3] += 1e-3;
  }
  long long t1 = clock64();
  if (lane == 0) cyc[1] = (t1 - t0) / iters;
  out[lane] = acc;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 16);
  k<<<1, 32>>>(o, c, 1000); k2<<<1, 32>>>(o, c, 1000); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, c, 10000); k2<<<1, 32>>>(o, c, 10000); cudaDeviceSynchronize();
  long long h[2]; cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
  printf("{\"dump_sync_lds_cycles\": %lld, \"select_shfl_cycles\": %lld}\n", h[0], h[1]);
}
