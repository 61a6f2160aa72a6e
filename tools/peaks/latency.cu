// Dependent-chain latencies (cycles) of the instructions on the FFS draw's critical path:
// DFMA, DADD, DMUL, double reciprocal (1.0/x), SHFL (32-bit), LDS.64, and a shfl.up fp64 scan
// level. One warp, clock64 around N dependent operations.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 1024;

__global__ void lat(double* out, long long* cyc, double a, double b, int k) {
  __shared__ double sm[64];
  if (threadIdx.x < 64) sm[threadIdx.x] = threadIdx.x * 1e-3;
  __syncthreads();
  double x = a + threadIdx.x * 1e-9;
  long long t0, t1;
  // DFMA
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = fma(x, b, a);
  t1 = clock64();
  cyc[0] = t1 - t0;
  // DADD
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = x + b;
  t1 = clock64();
  cyc[1] = t1 - t0;
  // DMUL
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = x * b;
  t1 = clock64();
  cyc[2] = t1 - t0;
  // reciprocal
  double y = x + 1.5;
  t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N / 8; ++i) y = 1.0 / y + 1.0;
  t1 = clock64();
  cyc[3] = (t1 - t0) * 8;
  // SHFL
  int v = threadIdx.x + k;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) v = __shfl_sync(0xffffffffu, v, (threadIdx.x + 1) & 31);
  t1 = clock64();
  cyc[4] = t1 - t0;
  // LDS (pointer chase through smem index)
  int idx = threadIdx.x & 7;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) idx = ((int)(sm[idx] * 1000.0) + 1) & 31;
  t1 = clock64();
  cyc[5] = t1 - t0;
  // fp64 scan level: shfl.up x2 + predicated add
  double s = x;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) {
    double t = __shfl_up_sync(0xffffffffu, s, 1);
    s = (threadIdx.x >= 1) ? s + t * 1e-300 : s;
  }
  t1 = clock64();
  cyc[6] = t1 - t0;
  // DSETP + vote (ballot) dependent chain
  unsigned m = threadIdx.x;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) m = __ballot_sync(0xffffffffu, (double)m * b > a) ^ threadIdx.x;
  t1 = clock64();
  cyc[7] = t1 - t0;
  out[threadIdx.x] = x + y + v + idx + s + m;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 64 * 8);
  cudaMalloc(&cyc, 16 * 8);
  lat<<<1, 32>>>(out, cyc, 1e-3, 0.999, 0);
  lat<<<1, 32>>>(out, cyc, 1e-3, 0.999, 0);
  cudaDeviceSynchronize();
  long long h[16];
  cudaMemcpy(h, cyc, 16 * 8, cudaMemcpyDeviceToHost);
  const char* names[] = {"dfma", "dadd", "dmul", "drcp(1/x)+dadd", "shfl32", "lds64+cvt chain", "fp64 scan level", "dsetp+ballot"};
  printf("{");
  for (int i = 0; i < 8; ++i) printf("%s\"%s\": %.1f", i ? ", " : "", names[i], (double)h[i] / N);
  printf("}\n");
  return 0;
}
