// Single-warp FP64 issue rate (development): cycles per warp-instruction for independent DFMAs
// (32 accumulators) and for DMMA m8n8k4 (8 accumulator fragments), with 1..4 warps per
// scheduler (blockDim = 32 * 4 * k so that every SM sub-partition holds k warps).
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 2048;

__global__ void dfma_rate(double* out, long long* cyc, double a, double b) {
  double acc[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = fma(acc[i], a, b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if ((threadIdx.x & 31) == 0) cyc[threadIdx.x >> 5] = (t1 - t0);
}

__global__ void dmma_rate(double* out, long long* cyc, double a) {
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = threadIdx.x * 1e-3 + i;
  double av = a + threadIdx.x * 1e-6, bv = a - threadIdx.x * 1e-6;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS / 8; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(av), "d"(bv));
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if ((threadIdx.x & 31) == 0) cyc[threadIdx.x >> 5] = (t1 - t0);
}

int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 1 << 20);
  cudaMalloc(&c, 64 * 8);
  printf("{");
  for (int k = 1; k <= 4; ++k) {
    const int threads = 32 * 4 * k;
    dfma_rate<<<1, threads>>>(o, c, 0.999, 1e-3);
    dfma_rate<<<1, threads>>>(o, c, 0.999, 1e-3);
    cudaDeviceSynchronize();
    long long h[64];
    cudaMemcpy(h, c, 64 * 8, cudaMemcpyDeviceToHost);
    // cycles per DFMA warp-instruction per warp, and SMSP pipe cycles per DFMA
    const double per = (double)h[0] / (ITERS * 32.0);
    printf("%s\"dfma_cycles_per_instr_%dwarps_per_smsp\": %.2f", k > 1 ? ", " : "", k, per);
    dmma_rate<<<1, threads>>>(o, c, 0.5);
    dmma_rate<<<1, threads>>>(o, c, 0.5);
    cudaDeviceSynchronize();
    cudaMemcpy(h, c, 64 * 8, cudaMemcpyDeviceToHost);
    printf(", \"dmma_cycles_per_instr_%dwarps_per_smsp\": %.2f", k, (double)h[0] / (ITERS));
  }
  printf("}\n");
  return 0;
}
