// FP64 / on-chip bandwidth microbenchmarks for the roofline denominators of the
// FFS hot path (SURVEY.md §7 step 1 "B0 measure the box"). MEASURED_PEAKS.json
// carries HBM and bf16 only; this program measures, on one B200:
//   dfma   : FP64 FMA (DFMA) throughput, register operands, many independent chains
//   dmma   : FP64 tensor MMA (mma.sync.m8n8k4.f64 -> DMMA.8x8x4) throughput
//   lds64  : shared-memory load bandwidth with 8-byte per-lane, conflict-free loads
//   l2rd   : read bandwidth of a buffer that fits in L2 (re-read many times)
// Output: one JSON object on stdout.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peaks fp64_peaks.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int kChains = 8;

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c];
  if (s == 1234.5) out[0] = s;  // never true; keeps the chains live
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-12, b = 0.999999;
  double c[kChains][2];
#pragma unroll
  for (int t = 0; t < kChains; ++t) { c[t][0] = 0; c[t][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < kChains; ++t) {
      asm volatile(
          "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
          : "+d"(c[t][0]), "+d"(c[t][1])
          : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < kChains; ++t) s += c[t][0] + c[t][1];
  if (s == 1234.5) out[0] = s;
}

__global__ void lds_kernel(double* out, int iters) {
  extern __shared__ double sm[];
  const int n = 4096;  // 32 KB
  for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = i * 1e-3;
  __syncthreads();
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  int base = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    int o = (i * 128) & (n - 1);
    s0 += sm[(base + o) & (n - 1)];
    s1 += sm[(base + o + 1024) & (n - 1)];
    s2 += sm[(base + o + 2048) & (n - 1)];
    s3 += sm[(base + o + 3072) & (n - 1)];
  }
  double s = s0 + s1 + s2 + s3;
  if (s == 1234.5) out[0] = s;
}

__global__ void l2rd_kernel(const double2* __restrict__ buf, size_t n2, int reps, double* out) {
  double acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride) {
      double2 v = __ldcg(buf + i);
      acc += v.x + v.y;
    }
  if (acc == 1234.5) out[0] = acc;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  double* out;
  CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float ms;

  // DFMA: 2 flops per fma
  {
    int threads = 256, blocks = sms * 8, iters = 1 << 15;
    dfma_kernel<<<blocks, threads>>>(out, 64, 0.999, 1e-7);
    CK(cudaDeviceSynchronize());
    double best = 0;
    for (int rep = 0; rep < 5; ++rep) {
      CK(cudaEventRecord(e0));
      dfma_kernel<<<blocks, threads>>>(out, iters, 0.999, 1e-7);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
      double tf = 2.0 * kChains * (double)iters * threads * blocks / (ms * 1e-3) / 1e12;
      if (tf > best) best = tf;
    }
    printf("{\"sms\": %d, \"smem_per_sm\": %zu, \"smem_per_block_optin\": %zu, \"l2_bytes\": %d, "
           "\"regs_per_sm\": %d, \"clock_khz\": %d,\n", sms, p.sharedMemPerMultiprocessor,
           p.sharedMemPerBlockOptin, p.l2CacheSize, p.regsPerMultiprocessor, p.clockRate);
    printf(" \"dfma_tflops\": %.3f,\n", best);
  }
  // DMMA m8n8k4: 2*8*8*4 = 512 flops per warp-instruction
  {
    int threads = 256, blocks = sms * 8, iters = 1 << 13;
    dmma_kernel<<<blocks, threads>>>(out, 64);
    CK(cudaDeviceSynchronize());
    double best = 0;
    for (int rep = 0; rep < 5; ++rep) {
      CK(cudaEventRecord(e0));
      dmma_kernel<<<blocks, threads>>>(out, iters);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
      double tf = 512.0 * kChains * (double)iters * (threads / 32) * blocks / (ms * 1e-3) / 1e12;
      if (tf > best) best = tf;
    }
    printf(" \"dmma_tflops\": %.3f,\n", best);
  }
  // shared memory LDS.64 bandwidth (bytes/clk/SM reported from the SM clock we cannot read here;
  // report GB/s per SM and total)
  {
    int threads = 512, blocks = sms * 4, iters = 1 << 14;
    CK(cudaFuncSetAttribute(lds_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768));
    lds_kernel<<<blocks, threads, 32768>>>(out, 64);
    CK(cudaDeviceSynchronize());
    double best = 0;
    for (int rep = 0; rep < 5; ++rep) {
      CK(cudaEventRecord(e0));
      lds_kernel<<<blocks, threads, 32768>>>(out, iters);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
      double gbs = 4.0 * 8.0 * (double)iters * threads * blocks / (ms * 1e-3) / 1e9;
      if (gbs > best) best = gbs;
    }
    printf(" \"lds64_gbs_total\": %.1f, \"lds64_gbs_per_sm\": %.1f,\n", best, best / sms);
  }
  // L2-resident read bandwidth: 32 MB buffer re-read
  {
    size_t bytes = 32u << 20;
    double2* buf;
    CK(cudaMalloc(&buf, bytes));
    CK(cudaMemset(buf, 0, bytes));
    size_t n2 = bytes / 16;
    int threads = 512, blocks = sms * 4, reps = 20;
    l2rd_kernel<<<blocks, threads>>>(buf, n2, 2, out);
    CK(cudaDeviceSynchronize());
    double best = 0;
    for (int rep = 0; rep < 5; ++rep) {
      CK(cudaEventRecord(e0));
      l2rd_kernel<<<blocks, threads>>>(buf, n2, reps, out);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
      double gbs = (double)bytes * reps / (ms * 1e-3) / 1e9;
      if (gbs > best) best = gbs;
    }
    printf(" \"l2_read_gbs_32MB\": %.1f}\n", best);
    CK(cudaFree(buf));
  }
  return 0;
}
