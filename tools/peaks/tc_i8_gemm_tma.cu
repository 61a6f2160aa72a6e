// Prototype (round-2 groundwork), TMA variant of tc_i8_gemm.cu: an INT8 GEMM on the 5th-generation tensor cores
// (tcgen05.mma.kind::i8, accumulator in TMEM), the building block of an Ozaki-style FP64
// emulation of the dense path's P = U Y. Not used by libffs.
//   C[M][N] (int32, row-major) = A[M][K] (int8, row-major) * B[N][K]^T (int8, row-major = K-major)
// CTA tile 128 x 256, K staged 128 bytes at a time (four tcgen05.mma of K = 32), 3-stage cp.async
// ring into the canonical no-swizzle K-major layout (8-row x 16-byte core matrices); producer warps
// and one MMA-issuing thread hand stages over through full/empty mbarriers; 4 warps read the
// accumulator back with tcgen05.ld. Checks 512 x 512 x 1024 against the host, then times 8192^3.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_i8_gemm tc_i8_gemm.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include <cuda.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int BM = 128, BN = 256, BK = 128, STAGES = 4, THREADS = 256;
constexpr int TILE_A = BM * BK, TILE_B = BN * BK;  // bytes per stage

__device__ __forceinline__ unsigned sm_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

// canonical K-major, no swizzle: core matrix (row group g = r/8, 16-byte K chunk c) at
// (g * (BK/16) + c) * 128 bytes, row r%8 at +16*(r%8). LBO (K-adjacent cores) = 128 B,
// SBO (8-row-adjacent cores) = (BK/16) * 128 B.
__device__ __forceinline__ int core_off(int r, int c) { return ((r >> 3) * (BK / 16) + c) * 128 + (r & 7) * 16; }

// K-major, 128-byte swizzle (what TMA writes with CU_TENSOR_MAP_SWIZZLE_128B): 8-row x 128-byte
// atoms, SBO = 1024 B between atoms along M/N; the K = 32-byte slice ks of the 128-byte rows is
// addressed by advancing the start address by 32 B (the hardware applies the XOR swizzle).
__device__ __forceinline__ uint64_t smem_desc(const void* base) {
  const uint64_t addr = sm_u32(base);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFF;                          // start address [0,14)
  d |= (uint64_t)1 << 16;                             // leading byte offset (unused for SW128 K-major)
  d |= (uint64_t)((1024 >> 4) & 0x3FFF) << 32;        // stride byte offset [32,46)
  d |= (uint64_t)1 << 46;                             // version (sm100)
  d |= (uint64_t)2 << 61;                             // layout type SWIZZLE_128B
  return d;
}

// kind::i8 instruction descriptor: D s32, A s8, B s8, both K-major, N = 128, M = 128
__device__ __forceinline__ uint32_t idesc_i8() {
  uint32_t d = 0;
  d |= 2u << 4;                // c_format S32
  d |= 1u << 7;                // a_format s8
  d |= 1u << 10;               // b_format s8
  d |= (uint32_t)(BN >> 3) << 17;
  d |= (uint32_t)(BM >> 4) << 24;
  return d;
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

// Warp-specialised: warps 4..7 load (cp.async, wait, proxy fence, arrive on full[st]); warp 0
// lane 0 waits full[st], issues BK/32 MMAs and commits them to empty[st]; the producers wait
// empty[st] before refilling it. Epilogue: warps 0..3 read TMEM lanes 32w..32w+31.
__global__ void __launch_bounds__(THREADS, 1) tc_i8_gemm(const __grid_constant__ CUtensorMap tmA,
                                                         const __grid_constant__ CUtensorMap tmB,
                                                         int32_t* __restrict__ C, int M, int N, int K) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sa = smem;                                 // [STAGES][TILE_A]
  unsigned char* sb = smem + STAGES * TILE_A;               // [STAGES][TILE_B]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * (TILE_A + TILE_B));
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int KT = K / BK;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sm_u32(tmem_slot)), "r"(BN)
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

  if (warp == 4 && lane == 0) {  // TMA producer
    for (int kt = 0; kt < KT; ++kt) {
      const int st = kt % STAGES;
      if (kt >= STAGES) mbar_wait(empty + st, ((kt / STAGES) - 1) & 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm_u32(full + st)),
                   "r"(TILE_A + TILE_B)
                   : "memory");
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              sm_u32(sa + st * TILE_A)),
          "l"(&tmA), "r"(kt * BK), "r"(m0), "r"(sm_u32(full + st))
          : "memory");
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              sm_u32(sb + st * TILE_B)),
          "l"(&tmB), "r"(kt * BK), "r"(n0), "r"(sm_u32(full + st))
          : "memory");
    }
  } else if (warp == 0 && lane == 0) {  // MMA issuer
    const uint32_t idesc = idesc_i8();
    for (int kt = 0; kt < KT; ++kt) {
      const int st = kt % STAGES;
      mbar_wait(full + st, (kt / STAGES) & 1);  // TMA bytes landed (async proxy: no fence needed)
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int ks = 0; ks < BK / 32; ++ks) {
        const uint64_t da = smem_desc(sa + st * TILE_A + ks * 32);
        const uint64_t db = smem_desc(sb + st * TILE_B + ks * 32);
        const uint32_t acc = (kt > 0 || ks > 0) ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(da), "l"(db), "r"(idesc), "r"(acc)
            : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sm_u32(empty + st))
                   : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sm_u32(done))
                 : "memory");
  }
  if (warp < 4) {
    mbar_wait(done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int row = m0 + warp * 32 + lane;
#pragma unroll 1
    for (int cb = 0; cb < BN; cb += 32) {
      uint32_t v[32];
      const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + cb;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
            "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
            "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (row < M) {
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<int4*>(C + (size_t)row * N + n0 + cb + j) =
              make_int4((int)v[j], (int)v[j + 1], (int)v[j + 2], (int)v[j + 3]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN) : "memory");
}

static size_t smem_bytes() { return STAGES * (TILE_A + TILE_B) + (2 * STAGES + 1) * 8 + 16 + 1024; }

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
  const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)K};
  const cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  const cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { fprintf(stderr, "cuTensorMapEncodeTiled failed %d\n", (int)r); exit(1); }
  return m;
}

static double run(int M, int N, int K, bool check) {
  std::vector<int8_t> ha((size_t)M * K), hb((size_t)N * K);
  unsigned s = 12345;
  for (auto& x : ha) { s = s * 1103515245u + 12345u; x = (int8_t)((s >> 16) % 255 - 127); }
  for (auto& x : hb) { s = s * 1103515245u + 12345u; x = (int8_t)((s >> 16) % 255 - 127); }
  int8_t *da, *db;
  int32_t* dc;
  CK(cudaMalloc(&da, ha.size()));
  CK(cudaMalloc(&db, hb.size()));
  CK(cudaMalloc(&dc, (size_t)M * N * 4));
  CK(cudaMemcpy(da, ha.data(), ha.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db, hb.data(), hb.size(), cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(tc_i8_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes()));
  dim3 grid(N / BN, M / BM);
  const CUtensorMap ta = make_map(da, M, K, BM), tb = make_map(db, N, K, BN);
  tc_i8_gemm<<<grid, THREADS, smem_bytes()>>>(ta, tb, dc, M, N, K);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  double tops = 0;
  if (check) {
    std::vector<int32_t> hc((size_t)M * N);
    CK(cudaMemcpy(hc.data(), dc, hc.size() * 4, cudaMemcpyDeviceToHost));
    long bad = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        long ref = 0;
        for (int k = 0; k < K; ++k) ref += (long)ha[(size_t)i * K + k] * hb[(size_t)j * K + k];
        if (ref != hc[(size_t)i * N + j]) {
          if (bad < 5) fprintf(stderr, "mismatch C[%d][%d] = %d, ref %ld\n", i, j, hc[(size_t)i * N + j], ref);
          ++bad;
        }
      }
    printf("{\"check\": \"%s\", \"M\": %d, \"N\": %d, \"K\": %d, \"mismatches\": %ld}\n", bad ? "FAIL" : "ok", M, N, K, bad);
  } else {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      tc_i8_gemm<<<grid, THREADS, smem_bytes()>>>(ta, tb, dc, M, N, K);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    tops = 2.0 * M * N * (double)K / (best * 1e-3) / 1e12;
    printf("{\"tc_i8_gemm_tops\": %.1f, \"M\": %d, \"N\": %d, \"K\": %d, \"ms\": %.3f}\n", tops, M, N, K, best);
  }
  cudaFree(da);
  cudaFree(db);
  cudaFree(dc);
  return tops;
}

int main() {
  run(512, 512, 1024, true);
  run(8192, 8192, 8192, false);
  run(16384, 8192, 1024, false);  // the C5 dense block's shape (one slice pair): M = L, N = 8 S, K = N
  run(4096, 16384, 2048, false);  // C4 (complex as real 2N)
  return 0;
}
