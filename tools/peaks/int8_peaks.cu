// INT8 tensor throughput on B200 for the Ozaki-style FP64-emulation question:
//   imma : legacy mma.sync.m16n8k32.s8.s8.s32 (what a non-tcgen05 kernel can issue), many
//          independent accumulators per warp, 8 warps per SM x 4 CTAs
// torch._int_mm (cuBLASLt, tcgen05) is timed by the driver script for the tcgen05 reference.
// Output: one JSON object on stdout.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int kAcc = 8;

__global__ void imma_kernel(int* out, int iters) {
  unsigned a0 = 0x01020304u + threadIdx.x, a1 = 0x05060708u, a2 = 0x0a0b0c0du, a3 = 0x01010101u;
  unsigned b0 = 0x02020202u, b1 = 0x03030303u + threadIdx.x;
  int c[kAcc][4];
#pragma unroll
  for (int t = 0; t < kAcc; ++t) c[t][0] = c[t][1] = c[t][2] = c[t][3] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < kAcc; ++t)
      asm volatile(
          "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
          : "+r"(c[t][0]), "+r"(c[t][1]), "+r"(c[t][2]), "+r"(c[t][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  int s = 0;
#pragma unroll
  for (int t = 0; t < kAcc; ++t) s += c[t][0] + c[t][1] + c[t][2] + c[t][3];
  if (s == 12345) out[0] = s;
}

int main() {
  int dev = 0, sms = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  int* out;
  CK(cudaMalloc(&out, 64));
  const int iters = 4096, threads = 256, blocks = sms * 4;
  imma_kernel<<<blocks, threads>>>(out, 16);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    imma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double ops = 2.0 * 16 * 8 * 32 * (double)kAcc * iters * (blocks * threads / 32);
  printf("{\"imma_mma_sync_tops\": %.1f, \"sms\": %d}\n", ops / (best * 1e-3) / 1e12, sms);
  return 0;
}
