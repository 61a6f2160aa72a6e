// Prototype (round-2 groundwork): FP64 GEMM C = A B emulated on the INT8 tensor
// cores (Ozaki-style splitting), the candidate replacement of the dense path's DMMA GEMM.
//   A [M][K] fp64: row r scaled by 2^-ea[r] (|.| < 1), split into S signed 7-bit slices A_i
//   B [K][N] fp64: column c scaled by 2^-eb[c], split into S slices B_j (stored K-major: [N][K])
//   C = 2^(ea + eb) * sum_{i + j < S} 2^(-7 (i + j + 2)) A_i B_j
// One CTA computes a 128 x 64 tile: the S partial sums D_d = sum_{i + j = d} A_i B_j (exact in
// int32) live in S TMEM accumulators of 64 columns; per 64-byte K chunk one thread issues the
// TMA loads of every slice (3-D tensor maps [S][rows][K], 64-byte swizzle) and one thread issues
// the S (S + 1) / 2 x 2 tcgen05.mma.kind::i8; the epilogue converts and scales in fp64.
// Checks against a host fp64 GEMM, then times the C5 dense-block shape.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ozaki_gemm ozaki_gemm.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int S = 7;                     // slices
constexpr int BM = 128, BN = 64, BK = 64, STAGES = 2, THREADS = 192;
constexpr int TA = BM * BK, TB = BN * BK;  // bytes per slice per stage
constexpr int STAGE_BYTES = S * (TA + TB);

__device__ __forceinline__ unsigned sm_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

// K-major, 64-byte swizzle: 8-row x 64-byte atoms, SBO = 512 B; K slice ks at +32 B
__device__ __forceinline__ uint64_t smem_desc(const void* base) {
  const uint64_t addr = sm_u32(base);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFF;
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((512 >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;  // SWIZZLE_64B
  return d;
}
__device__ __forceinline__ uint32_t idesc_i8() {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sm_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n\t}" ::"r"(sm_u32(b)),
      "r"(parity)
      : "memory");
}

__global__ void __launch_bounds__(THREADS, 1) ozaki_gemm(const __grid_constant__ CUtensorMap tmA,
                                                         const __grid_constant__ CUtensorMap tmB,
                                                         const int* __restrict__ ea, const int* __restrict__ eb,
                                                         double* __restrict__ C, int M, int N, int K) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int KT = K / BK;
  constexpr int TCOLS = 512;  // S x 64 <= 512 columns

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sm_u32(tmem_slot)), "r"(TCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (t == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 4 && lane == 0) {  // TMA producer: every slice of A and B for this K chunk
    for (int kt = 0; kt < KT; ++kt) {
      const int st = kt % STAGES;
      if (kt >= STAGES) mbar_wait(empty + st, ((kt / STAGES) - 1) & 1);
      unsigned char* sbase = smem + st * STAGE_BYTES;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm_u32(full + st)), "r"(STAGE_BYTES)
                   : "memory");
#pragma unroll
      for (int i = 0; i < S; ++i) {
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                sm_u32(sbase + i * TA)),
            "l"(&tmA), "r"(kt * BK), "r"(m0), "r"(i), "r"(sm_u32(full + st))
            : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                sm_u32(sbase + S * TA + i * TB)),
            "l"(&tmB), "r"(kt * BK), "r"(n0), "r"(i), "r"(sm_u32(full + st))
            : "memory");
      }
    }
  } else if (warp == 5 && lane == 0) {  // MMA issuer
    const uint32_t idesc = idesc_i8();
    for (int kt = 0; kt < KT; ++kt) {
      const int st = kt % STAGES;
      mbar_wait(full + st, (kt / STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const unsigned char* sbase = smem + st * STAGE_BYTES;
#pragma unroll
      for (int i = 0; i < S; ++i)
#pragma unroll
        for (int j = 0; j < S - i; ++j) {
          const uint32_t dcol = tmem + (uint32_t)((i + j) * BN);
#pragma unroll
          for (int ks = 0; ks < BK / 32; ++ks) {
            const uint64_t da = smem_desc(sbase + i * TA + ks * 32);
            const uint64_t db = smem_desc(sbase + S * TA + j * TB + ks * 32);
            const uint32_t acc = (kt > 0 || ks > 0 || i > 0) ? 1u : 0u;  // first write of D_{i+j}: i = 0
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "setp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(dcol),
                "l"(da), "l"(db), "r"(idesc), "r"(acc)
                : "memory");
          }
        }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sm_u32(empty + st))
                   : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sm_u32(done))
                 : "memory");
  }
  if (warp < 4) {  // epilogue: row warp*32 + lane of the tile, 64 columns in fp64
    mbar_wait(done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    double acc[BN];
#pragma unroll
    for (int c = 0; c < BN; ++c) acc[c] = 0.0;
#pragma unroll
    for (int d = S - 1; d >= 0; --d) {  // smallest terms first
      const double sc = ldexp(1.0, -7 * (d + 2));
#pragma unroll
      for (int cb = 0; cb < BN; cb += 32) {
        uint32_t v[32];
        const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(d * BN + cb);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int c = 0; c < 32; ++c) acc[cb + c] = fma((double)(int)v[c], sc, acc[cb + c]);
      }
    }
    const int row = m0 + warp * 32 + lane;
    if (row < M) {
      const double sr = ldexp(1.0, ea[row]);
#pragma unroll
      for (int c = 0; c < BN; c += 2) {
        const int col = n0 + c;
        *reinterpret_cast<double2*>(C + (size_t)row * N + col) =
            make_double2(acc[c] * sr * ldexp(1.0, eb[col]), acc[c + 1] * sr * ldexp(1.0, eb[col + 1]));
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS) : "memory");
}

// ---- host: splitting, tensor maps, check, timing
static void split_rows(const std::vector<double>& X, int rows, int K, bool transposeKN, std::vector<int8_t>& sl,
                       std::vector<int>& e) {
  // X is rows x K (row-major) when !transposeKN; K x rows (row-major) when transposeKN (columns
  // of a K x N matrix become the K-major rows of the slices)
  sl.assign((size_t)S * rows * K, 0);
  e.assign(rows, 0);
  for (int r = 0; r < rows; ++r) {
    double mx = 0;
    for (int k = 0; k < K; ++k) mx = std::max(mx, std::fabs(transposeKN ? X[(size_t)k * rows + r] : X[(size_t)r * K + k]));
    int ex = 0;
    if (mx > 0) std::frexp(mx, &ex);  // mx = f 2^ex, f in [0.5, 1): |x / 2^ex| < 1
    e[r] = ex;
    for (int k = 0; k < K; ++k) {
      double v = std::ldexp(transposeKN ? X[(size_t)k * rows + r] : X[(size_t)r * K + k], -ex);
      for (int i = 0; i < S; ++i) {
        const double q = std::trunc(v * 128.0);
        sl[((size_t)i * rows + r) * K + k] = (int8_t)q;
        v = v * 128.0 - q;
      }
    }
  }
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static CUtensorMap make_map(const int8_t* ptr, int rows, int K, int box_rows) {
  static EncodeTiled enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q));
  }
  CUtensorMap m;
  const cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)S};
  const cuuint64_t strides[2] = {(cuuint64_t)K, (cuuint64_t)K * rows};
  const cuuint32_t box[3] = {(cuuint32_t)BK, (cuuint32_t)box_rows, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { fprintf(stderr, "cuTensorMapEncodeTiled failed %d\n", (int)r); exit(1); }
  return m;
}

static size_t smem_bytes() { return STAGES * STAGE_BYTES + (2 * STAGES + 1) * 8 + 16 + 1024; }

static void run(int M, int N, int K, bool check) {
  std::vector<double> A((size_t)M * K), B((size_t)K * N);
  unsigned s = 777;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return ((s >> 8) & 0xFFFFFF) / 16777216.0 - 0.5; };
  for (int r = 0; r < M; ++r) {
    const double sc = std::ldexp(1.0, (r % 7) - 3);  // rows of different magnitude
    for (int k = 0; k < K; ++k) A[(size_t)r * K + k] = rnd() * sc;
  }
  for (int k = 0; k < K; ++k)
    for (int c = 0; c < N; ++c) B[(size_t)k * N + c] = rnd() * std::ldexp(1.0, (c % 5) - 2);
  std::vector<int8_t> As, Bs;
  std::vector<int> ea, eb;
  split_rows(A, M, K, false, As, ea);
  split_rows(B, N, K, true, Bs, eb);
  int8_t *dA, *dB;
  int *dea, *deb;
  double* dC;
  CK(cudaMalloc(&dA, As.size()));
  CK(cudaMalloc(&dB, Bs.size()));
  CK(cudaMalloc(&dea, M * 4));
  CK(cudaMalloc(&deb, N * 4));
  CK(cudaMalloc(&dC, (size_t)M * N * 8));
  CK(cudaMemcpy(dA, As.data(), As.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, Bs.data(), Bs.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dea, ea.data(), M * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(deb, eb.data(), N * 4, cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(ozaki_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes()));
  const CUtensorMap ta = make_map(dA, M, K, BM), tb = make_map(dB, N, K, BN);
  dim3 grid(N / BN, M / BM);
  ozaki_gemm<<<grid, THREADS, smem_bytes()>>>(ta, tb, dea, deb, dC, M, N, K);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  if (check) {
    std::vector<double> hc((size_t)M * N);
    CK(cudaMemcpy(hc.data(), dC, hc.size() * 8, cudaMemcpyDeviceToHost));
    double maxrel = 0;  // error relative to sum_k |a_rk| |b_kc| (the scale of the dot product)
    for (int r = 0; r < M; ++r)
      for (int c = 0; c < N; ++c) {
        long double ref = 0, mag = 0;
        for (int k = 0; k < K; ++k) {
          ref += (long double)A[(size_t)r * K + k] * B[(size_t)k * N + c];
          mag += std::fabs(A[(size_t)r * K + k] * B[(size_t)k * N + c]);
        }
        const double rel = (double)(std::fabs((long double)hc[(size_t)r * N + c] - ref) / mag);
        maxrel = std::max(maxrel, rel);
      }
    printf("{\"check\": \"%s\", \"M\": %d, \"N\": %d, \"K\": %d, \"slices\": %d, \"max_err_rel_to_abs_dot\": %.3e}\n",
           maxrel < 1e-12 ? "ok" : "FAIL", M, N, K, S, maxrel);
  } else {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      ozaki_gemm<<<grid, THREADS, smem_bytes()>>>(ta, tb, dea, deb, dC, M, N, K);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    printf("{\"ozaki_fp64_equiv_tflops\": %.1f, \"M\": %d, \"N\": %d, \"K\": %d, \"slices\": %d, \"ms\": %.3f}\n",
           2.0 * M * N * (double)K / (best * 1e-3) / 1e12, M, N, K, S, best);
  }
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dea);
  cudaFree(deb);
  cudaFree(dC);
}

int main() {
  run(256, 128, 1024, true);
  run(16384, 8192, 1024, false);  // the C5 dense block (DMMA GEMM: 8.4 ms)
  run(4096, 16384, 2048, false);  // C4 (complex as real 2N; DMMA GEMM: 4.2 ms)
  return 0;
}
