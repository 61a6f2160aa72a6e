// C ABI of libffs.so (declarations and contracts: include/ffs.h).
// Argument validation, kernel-variant dispatch, workspace carving and the host-buffer path.
// No torch types, no hidden allocations; everything runs in the kernels of ffs_kernel.cuh.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <algorithm>

#include "ffs.h"
#include "ffs_kernel.cuh"
#include "ffs_warp_kernel.cuh"
#include "ffs_cluster_kernel.cuh"
#include "ffs_mma_kernel.cuh"
#include "ffs_dense.cuh"
#include "ffs_kptr.h"

namespace {

thread_local char g_err[512] = "";
thread_local int g_launches = 0;

// Optional CUDA-event timing of the dominant (sampling) kernel of each call, on the launch stream.
thread_local bool g_prof = false;
thread_local cudaEvent_t g_ev0 = nullptr, g_ev1 = nullptr;
thread_local bool g_ev_pending = false;
unsigned long long* g_timing = nullptr;  // development: device counters for FFS_DEBUG_SKIP bit3

cudaError_t launch_timed(const void* fn, dim3 grid, dim3 block, void** args, size_t smem, cudaStream_t s) {
  if (g_prof) {
    if (!g_ev0) {
      cudaEventCreate(&g_ev0);
      cudaEventCreate(&g_ev1);
    }
    cudaEventRecord(g_ev0, s);
  }
  cudaError_t e = cudaLaunchKernel(fn, grid, block, args, smem, s);
  if (g_prof && e == cudaSuccess) {
    cudaEventRecord(g_ev1, s);
    g_ev_pending = true;
  }
  return e;
}

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

constexpr size_t kAlign = 256;
size_t align_up(size_t v) { return (v + kAlign - 1) & ~(kAlign - 1); }

// ------------------------------------------------------------------ variant table
// A variant is a kernel instantiation ffs_sample_kernel<T, WARP, R, B, USMEM>.
struct Variant {
  bool warp;      // owner = one warp (true) or one CTA of G threads (false)
  int R, B;       // rows per thread, panel width
  bool usmem;     // U^T held in shared memory (shared by all owners of a CTA)
  int maxt;       // __launch_bounds__ of the instantiation
  const void* fn; // kernel
};

// warp-owner kernels: up to kWarpMaxThreads threads (= owners x 32) per CTA
constexpr int kWarpMaxThreads = 320;

template <typename T, bool WARP, int R, int B, bool USMEM, int MAXT = kWarpMaxThreads>
Variant make_variant() {
  return Variant{WARP, R, B, USMEM, MAXT,
                 ffsk::sample_kernel_ptr<T, WARP, R, B, USMEM, MAXT>()};
}

constexpr size_t kMaxSmem = 227 * 1024;

struct Plan {
  Variant v;
  int es;              // scalar bytes
  int G;               // threads per owner
  int Lp;              // rows covered per owner
  int threads;         // blockDim.x
  int owners_per_cta;
  int grid;
  int ut_stride;
  size_t owner_smem, ushared_smem, smem;
  size_t ws_ut, ws_wfull;  // workspace bytes
};

bool pick_variant(int L, int N, int Np, int dtype, Variant& v) {
  const bool c = dtype == FFS_C128;
  const size_t es = c ? 16 : 8;
  // U^T in shared memory if the whole (padded) matrix takes <= 96 KB: one copy per CTA,
  // shared by all warp-owners of that CTA.
  auto fits = [&](int R) { return (size_t)N * (size_t)(32 * R + 2) * es <= 96 * 1024; };
  // Warp owners (L <= 256 real / 128 complex): panel R x B per lane in registers.
  // CTA owners: one sample per CTA; the L x B panel must fit the SM's register file, so B
  // shrinks as L grows (the large-L configs are register-capacity bound).
  if (!c) {
    if (L <= 32)  { v = fits(1) ? make_variant<double, true, 1, 8, true>() : make_variant<double, true, 1, 8, false>(); return true; }
    if (L <= 64)  { v = fits(2) ? make_variant<double, true, 2, 8, true>() : make_variant<double, true, 2, 8, false>(); return true; }
    if (L <= 128) { v = fits(4) ? make_variant<double, true, 4, 8, true>() : make_variant<double, true, 4, 8, false>(); return true; }
    if (L <= 256) { v = fits(8) ? make_variant<double, true, 8, 8, true, 256>() : make_variant<double, true, 8, 8, false, 256>(); return true; }
    if (L <= 1024)  { v = make_variant<double, false, 4, 8, false, 256>(); return true; }
    if (L <= 4096)  { v = make_variant<double, false, 4, 4, false, 1024>(); return true; }
    if (L <= 8192)  { v = make_variant<double, false, 8, 2, false, 1024>(); return true; }
    if (L <= 16384) { v = make_variant<double, false, 16, 1, false, 1024>(); return true; }
  } else {
    if (L <= 32)  { v = fits(1) ? make_variant<cplx, true, 1, 4, true>() : make_variant<cplx, true, 1, 4, false>(); return true; }
    if (L <= 64)  { v = fits(2) ? make_variant<cplx, true, 2, 4, true>() : make_variant<cplx, true, 2, 4, false>(); return true; }
    if (L <= 128) { v = fits(4) ? make_variant<cplx, true, 4, 4, true>() : make_variant<cplx, true, 4, 4, false>(); return true; }
    if (L <= 1024)  { v = make_variant<cplx, false, 4, 4, false, 256>(); return true; }
    if (L <= 4096)  { v = make_variant<cplx, false, 4, 2, false, 1024>(); return true; }
    if (L <= 8192)  { v = make_variant<cplx, false, 8, 1, false, 1024>(); return true; }
  }
  (void)Np;
  return false;
}

size_t owner_bytes(bool c, int B, int N, int Np) {
  if (c) {
    switch (B) {
      case 1: return ffsk::OwnerLayout<cplx, 1>(N, Np).total;
      case 2: return ffsk::OwnerLayout<cplx, 2>(N, Np).total;
      case 4: return ffsk::OwnerLayout<cplx, 4>(N, Np).total;
      default: return ffsk::OwnerLayout<cplx, 8>(N, Np).total;
    }
  }
  switch (B) {
    case 1: return ffsk::OwnerLayout<double, 1>(N, Np).total;
    case 2: return ffsk::OwnerLayout<double, 2>(N, Np).total;
    case 4: return ffsk::OwnerLayout<double, 4>(N, Np).total;
    default: return ffsk::OwnerLayout<double, 8>(N, Np).total;
  }
}

int make_plan(int64_t L, int64_t N, int64_t Np, int dtype, int64_t M, Plan& pl) {
  if (L < 1 || N < 1 || N > L || Np < 1 || Np > N || L > INT32_MAX || M < 0)
    return fail(FFS_EINVAL, "invalid shape L=%lld N=%lld N'=%lld M=%lld", (long long)L, (long long)N,
                (long long)Np, (long long)M);
  if (dtype != FFS_F64 && dtype != FFS_C128) return fail(FFS_EINVAL, "unknown dtype %d", dtype);
  if (!pick_variant((int)L, (int)N, (int)Np, dtype, pl.v))
    return fail(FFS_EINVAL, "unsupported L=%lld for dtype %d (max 16384)", (long long)L, dtype);
  const bool c = dtype == FFS_C128;
  pl.es = c ? 16 : 8;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(FFS_ECUDA, "cudaGetDevice failed");
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, pl.v.fn) != cudaSuccess) return fail(FFS_ECUDA, "cudaFuncGetAttributes failed");
  const int regs = std::max(fa.numRegs, 1);
  pl.owner_smem = owner_bytes(c, pl.v.B, (int)N, (int)Np);
  if (pl.v.warp) {
    pl.G = 32;
    pl.Lp = 32 * pl.v.R;
    pl.ut_stride = pl.Lp + (c ? 1 : 2);  // +16 B per column: spreads column bases over banks
    pl.ushared_smem = pl.v.usmem ? ffsk::align16((size_t)N * pl.ut_stride * pl.es) : 0;
    // warps per CTA: bounded by registers (one CTA per SM when U^T is shared), smem, and 16
    const int by_regs = std::max(1, 65536 / (((regs * 32 + 255) / 256) * 256));
    int w = std::min(pl.v.maxt / 32, by_regs);
    while (w > 1 && pl.ushared_smem + (size_t)w * pl.owner_smem > kMaxSmem) --w;
    if (!pl.v.usmem) w = std::min(w, 4);
    pl.owners_per_cta = w;
    pl.threads = 32 * w;
  } else {
    const int rows_per_warp = 32 * pl.v.R;
    const int warps = (int)((L + rows_per_warp - 1) / rows_per_warp);
    pl.G = 32 * warps;
    pl.Lp = pl.G * pl.v.R;
    pl.ut_stride = 0;
    pl.ushared_smem = 0;
    pl.owners_per_cta = 1;
    pl.threads = pl.G;
    if (pl.G > pl.v.maxt)
      return fail(FFS_EINVAL, "variant needs %d threads > %d", pl.G, pl.v.maxt);
  }
  pl.smem = pl.ushared_smem + (size_t)pl.owners_per_cta * pl.owner_smem;
  if (pl.smem > kMaxSmem) return fail(FFS_EINVAL, "shared memory %zu > %zu (N=%lld)", pl.smem, kMaxSmem, (long long)N);
  if (cudaFuncSetAttribute(pl.v.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem) != cudaSuccess)
    return fail(FFS_ECUDA, "cudaFuncSetAttribute(smem=%zu) failed", pl.smem);
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pl.v.fn, pl.threads, pl.smem) != cudaSuccess || per_sm < 1)
    return fail(FFS_EINVAL, "kernel does not fit on an SM (threads=%d smem=%zu regs=%d)", pl.threads, pl.smem, regs);
  const int64_t want = (M + pl.owners_per_cta - 1) / pl.owners_per_cta;
  pl.grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)per_sm * sms));
  pl.ws_ut = pl.v.usmem ? 0 : align_up((size_t)N * pl.Lp * pl.es);
  pl.ws_wfull = align_up((size_t)pl.grid * pl.owners_per_cta * (size_t)Np * Np * pl.es);
  return FFS_OK;
}

// ------------------------------------------------------------------ fast warp-owner path
// Real U, L <= 256, N' <= kMaxNpWarp, U^T small enough for shared memory: ffs_seg_kernel
// (one CTA per SM, G-lane segments of warps = sample owners) after ffs_permute_kernel.
struct WarpPlan {
  const void* fn;
  int R, B, S, G = 32, maxt, warps, grid, Lp, ut_stride;
  bool mma = false;  // ffs_mma_kernel (DMMA contraction, B = 8, its own U^T swizzle and slice)
  size_t ushared, owner, smem, ws_perm, ws_w = 0;
  int perm_tpb;
  size_t perm_smem;
};

template <int R, int B, int G, int MAXT, bool TIMING = false, int OPT = 0>
void warp_fn_seg(WarpPlan& w) {
  w.fn = ffsk::seg_kernel_ptr<R, B, G, MAXT, TIMING, OPT>();
  w.R = R;
  w.B = B;
  w.S = 32 / G;  // samples per warp (one per G-lane segment)
  w.G = G;
  w.maxt = MAXT;
}

bool warp_eligible(int64_t L, int64_t N, int64_t Np, int dtype) {
  if (dtype != FFS_F64 || L > 256 || Np > ffsk::kMaxNpWarp || N > 4096) return false;
  return (size_t)N * (256 + 2) * 8 <= 100 * 1024;  // padded U^T fits shared memory
}

int make_warp_plan(int64_t L, int64_t N, int64_t Np, int64_t M, WarpPlan& w) {
  const char* var = getenv("FFS_WARP_VARIANT");  // development: measured variants (profiles/)
  {
    // segmented kernel, OPT = 7 (+128 for G = 32): kept partial sums, pivot row through smem,
    // flat Gauss-Jordan, no warp vote when the segment is the whole warp
    // (variants measured in profiles/r01_ncu_summary.md; "base" = the first segmented kernel)
    const bool base = var && strcmp(var, "base") == 0;
    const size_t ush = ffsk::align16((size_t)N * (256 + 2) * 8);
    const bool fits16 = ush + 16 * ffsk::WarpLayout((int)Np, 4, true).total <= kMaxSmem;
    // L <= 16 (C1): 4-lane segments, 8 samples per warp (0.086 ms vs 0.092 ms with 8-lane segments)
    if (L <= 16) warp_fn_seg<4, 4, 4, 512, false, 7>(w);
    else if (L <= 32) warp_fn_seg<4, 4, 8, 512, false, 7>(w);
    else if (L <= 64) warp_fn_seg<8, 4, 8, 384, false, 7>(w);
    else if (L <= 128) warp_fn_seg<8, 4, 16, 384, false, 7>(w);
    else if (base) warp_fn_seg<8, 4, 32, 384, false, 0>(w);
    else if (var && strcmp(var, "o7_384") == 0) warp_fn_seg<8, 4, 32, 384, false, 7>(w);
    else if (var && strcmp(var, "b8") == 0) warp_fn_seg<8, 8, 32, 256, false, 7>(w);
    else if (var && strcmp(var, "o647") == 0) warp_fn_seg<8, 4, 32, 512, false, 647>(w);
    else if (var && strcmp(var, "t") == 0) warp_fn_seg<8, 4, 32, 512, true, 7>(w);  // phase timing
    else if (var && strncmp(var, "mma", 3) == 0) {
      const bool t256 = strcmp(var, "mma256") == 0;
      w.fn = t256 ? ffsk::mma_kernel_ptr<256>() : ffsk::mma_kernel_ptr<384>();
      w.R = 8;
      w.B = 8;
      w.S = 1;
      w.G = 32;
      w.maxt = t256 ? 256 : 384;
      w.mma = true;
    }
    else if (fits16) warp_fn_seg<8, 4, 32, 512, false, 135>(w);  // 16 owners/SM, 128 regs
    else warp_fn_seg<8, 4, 32, 384, false, 135>(w);              // 12 owners/SM (larger N')
  }
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(FFS_ECUDA, "cudaGetDevice failed");
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, w.fn) != cudaSuccess) return fail(FFS_ECUDA, "cudaFuncGetAttributes failed");
  w.Lp = w.G * w.R;
  w.ut_stride = w.mma ? ffsk::kMmaRows : w.Lp + 2;
  w.ushared = ffsk::align16((size_t)N * w.ut_stride * 8);
  w.owner = w.mma ? ffsk::MmaLayout((int)Np).total
                 : ffsk::WarpLayout((int)Np, w.B, true).total;  // per sample; a warp holds S slices
  // registers are allocated per SM sub-partition (4 x 16K); warps are spread round-robin
  const int by_regs = 4 * std::max(1, 16384 / (((std::max(fa.numRegs, 1) * 32 + 255) / 256) * 256));
  int warps = std::min(w.maxt / 32, by_regs);
  while (warps > 1 && w.ushared + (size_t)warps * w.S * w.owner > kMaxSmem) --warps;
  if (const char* fw = getenv("FFS_WARPS")) warps = std::max(1, std::min(warps, atoi(fw)));  // development
  w.warps = warps;
  w.smem = w.ushared + (size_t)warps * w.S * w.owner;
  if (w.smem > kMaxSmem) return fail(FFS_EINVAL, "warp path smem %zu too large", w.smem);
  const int64_t ctas = (M + (int64_t)warps * w.S - 1) / ((int64_t)warps * w.S);
  w.grid = (int)std::max<int64_t>(1, std::min<int64_t>(ctas, sms));
  w.ws_perm = align_up((size_t)std::max<int64_t>(M, 1) * Np * 4);
  w.perm_tpb = (int)std::max<int64_t>(1, std::min<int64_t>(128, 40960 / (4 * N)));
  w.perm_smem = (size_t)w.perm_tpb * N * 4;
  return FFS_OK;
}

int launch_warp(const void* U, int64_t L, int64_t N, int64_t M, int64_t Np, const double* uniforms,
                int32_t* positions, int32_t* flags, void* ws, size_t ws_bytes, cudaStream_t stream, int64_t S,
                double* trace) {
  WarpPlan w;
  int rc = make_warp_plan(L, N, Np, M, w);
  if (rc != FFS_OK) return rc;
  if (!ws || ws_bytes < w.ws_perm + w.ws_w)
    return fail(FFS_EINVAL, "workspace %zu bytes < required %zu", ws_bytes, w.ws_perm + w.ws_w);
  if (((uintptr_t)ws & (kAlign - 1)) != 0) return fail(FFS_EINVAL, "workspace not 256-byte aligned");
  int32_t* perm = static_cast<int32_t*>(ws);
  const int64_t pgrid = (M + w.perm_tpb - 1) / w.perm_tpb;
  ffsk::ffs_permute_kernel<<<(unsigned)pgrid, w.perm_tpb, w.perm_smem, stream>>>(uniforms, perm, M, (int)N, (int)Np);
  ++g_launches;
  if (cudaFuncSetAttribute(w.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)w.smem) != cudaSuccess)
    return fail(FFS_ECUDA, "cudaFuncSetAttribute(smem=%zu) failed", w.smem);
  ffsk::WarpParams p{};
  p.U = static_cast<const double*>(U);
  p.perm = perm;
  p.uniforms = uniforms;
  p.positions = positions;
  p.flags = flags;
  p.M = M;
  p.L = (int)L;
  p.N = (int)N;
  p.Np = (int)Np;
  p.Lp = w.Lp;
  p.ut_stride = w.ut_stride;
  p.ushared = w.ushared;
  p.owner_bytes = w.owner;
  p.wfull = nullptr;
  p.S = S > 0 ? std::min<int64_t>(S, M) : 0;
  p.trace = S > 0 ? trace : nullptr;
  const char* dbg = getenv("FFS_DEBUG_SKIP");  // development only: bits 0-2 break the results
  p.dbg = dbg ? atoi(dbg) : 0;
  p.timing = g_timing;
  void* args[] = {&p};
  cudaError_t e = launch_timed(w.fn, dim3(w.grid), dim3(32 * w.warps), args, w.smem, stream);
  if (e != cudaSuccess) return fail(FFS_ECUDA, "launch failed: %s", cudaGetErrorString(e));
  ++g_launches;
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(FFS_ECUDA, "CUDA error: %s", cudaGetErrorString(e));
  g_err[0] = 0;
  return FFS_OK;
}


// ------------------------------------------------------------------ cluster-owner path
// Large L (>= 2048): one thread-block cluster of CS CTAs per sample (ffs_cluster_kernel), the
// L x B panel spread over the cluster; B = 8.
struct ClusterPlan {
  const void* fn;
  int R, B, threads, CS, Lc, Lpt, grid, es;
  size_t smem, ws_ut, ws_w;
};

template <typename T, int R, int B, int MAXT>
void cluster_fn(ClusterPlan& c) {
  c.fn = ffsk::cluster_kernel_ptr<T, R, B, MAXT>();
  c.R = R;
  c.B = B;
  c.threads = MAXT;
}

bool cluster_eligible(int64_t L, int dtype) {
  const char* g = getenv("FFS_NO_CLUSTER");
  if (g && g[0] == '1') return false;
  return L >= 2048 && L <= (dtype == FFS_C128 ? 16 * 512 * 1 : 16 * 512 * 2);
}

int make_cluster_plan(int64_t L, int64_t N, int64_t Np, int dtype, int64_t M, ClusterPlan& c) {
  const bool cx = dtype == FFS_C128;
  const char* cv = getenv("FFS_CLUSTER_VARIANT");  // development: "b16" selects B=16 (slower)
  const bool b8 = !(cv && strcmp(cv, "b16") == 0);
  const bool t256 = cv && strcmp(cv, "t256") == 0;  // 256 threads x 2R rows (no spills; slower)
  if (cx) {
    if (!b8) cluster_fn<cplx, 1, 16, 512>(c);
    else if (t256) cluster_fn<cplx, 4, 8, 256>(c);
    else cluster_fn<cplx, 2, 8, 512>(c);
  } else {
    if (!b8) cluster_fn<double, 2, 16, 512>(c);
    else if (t256) cluster_fn<double, 8, 8, 256>(c);
    else cluster_fn<double, 4, 8, 512>(c);
  }
  c.es = cx ? 16 : 8;
  const int rows_per_cta = c.threads * c.R;
  c.CS = (int)((L + rows_per_cta - 1) / rows_per_cta);
  if (c.CS < 2) c.CS = 2;
  if (c.CS > 8) c.CS = 16;
  c.Lc = rows_per_cta;
  c.Lpt = c.CS * c.Lc;
  if (cx)
    c.smem = c.B == 8 ? ffsk::ClusterLayout<cplx, 8>((int)N, (int)Np, c.threads, c.R).total
                      : ffsk::ClusterLayout<cplx, 16>((int)N, (int)Np, c.threads, c.R).total;
  else
    c.smem = c.B == 8 ? ffsk::ClusterLayout<double, 8>((int)N, (int)Np, c.threads, c.R).total
                      : ffsk::ClusterLayout<double, 16>((int)N, (int)Np, c.threads, c.R).total;
  if (c.smem > kMaxSmem) return fail(FFS_EINVAL, "cluster path smem %zu > %zu (N'=%lld)", c.smem, kMaxSmem, (long long)Np);
  if (cudaFuncSetAttribute(c.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem) != cudaSuccess)
    return fail(FFS_ECUDA, "cudaFuncSetAttribute(smem) failed");
  if (c.CS > 8 && cudaFuncSetAttribute(c.fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
    return fail(FFS_ECUDA, "non-portable cluster size not allowed");
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = c.CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(c.threads);
  cfg.gridDim = dim3(c.CS);
  cfg.dynamicSmemBytes = c.smem;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int maxcl = 0;
  if (cudaOccupancyMaxActiveClusters(&maxcl, c.fn, &cfg) != cudaSuccess || maxcl < 1)
    return fail(FFS_EINVAL, "cluster of %d CTAs does not fit", c.CS);
  const int64_t ncl = std::max<int64_t>(1, std::min<int64_t>(M, maxcl));
  c.grid = (int)(ncl * c.CS);
  c.ws_ut = align_up((size_t)N * c.Lpt * c.es);
  c.ws_w = align_up((size_t)ncl * Np * Np * c.es);
  return FFS_OK;
}

int launch_cluster(const void* U, int64_t L, int64_t N, int dtype, int64_t M, int64_t Np, const double* uniforms,
                   int32_t* positions, int32_t* flags, void* ws, size_t ws_bytes, cudaStream_t stream, int64_t S,
                   double* trace) {
  ClusterPlan c;
  int rc = make_cluster_plan(L, N, Np, dtype, M, c);
  if (rc != FFS_OK) return rc;
  if (!ws || ws_bytes < c.ws_ut + c.ws_w)
    return fail(FFS_EINVAL, "workspace %zu bytes < required %zu", ws_bytes, c.ws_ut + c.ws_w);
  if (((uintptr_t)ws & (kAlign - 1)) != 0) return fail(FFS_EINVAL, "workspace not 256-byte aligned");
  char* w = static_cast<char*>(ws);
  ffsk::ClusterParams p{};
  p.U = static_cast<const double*>(U);
  p.Ut = reinterpret_cast<const double*>(w);
  p.L = (int)L;
  p.N = (int)N;
  p.Np = (int)Np;
  p.Lc = c.Lc;
  p.Lpt = c.Lpt;
  p.M = M;
  p.uniforms = uniforms;
  p.positions = positions;
  p.flags = flags;
  p.wfull = reinterpret_cast<double*>(w + c.ws_ut);
  p.S = S > 0 ? std::min<int64_t>(S, M) : 0;
  p.trace = S > 0 ? trace : nullptr;
  p.timing = g_timing;  // development (ffs_dev_timing); null unless enabled
  dim3 tb(32, 8), tg((unsigned)((c.Lpt + 31) / 32), (unsigned)((N + 31) / 32));
  if (dtype == FFS_C128)
    ffsk::transpose_pad_kernel<cplx><<<tg, tb, 0, stream>>>(p.U, const_cast<double*>(p.Ut), (int)L, (int)N, c.Lpt);
  else
    ffsk::transpose_pad_kernel<double><<<tg, tb, 0, stream>>>(p.U, const_cast<double*>(p.Ut), (int)L, (int)N, c.Lpt);
  ++g_launches;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = c.CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(c.threads);
  cfg.gridDim = dim3(c.grid);
  cfg.dynamicSmemBytes = c.smem;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* args[] = {&p};
  if (g_prof) {
    if (!g_ev0) {
      cudaEventCreate(&g_ev0);
      cudaEventCreate(&g_ev1);
    }
    cudaEventRecord(g_ev0, stream);
  }
  cudaError_t e = cudaLaunchKernelExC(&cfg, c.fn, args);
  if (e != cudaSuccess) return fail(FFS_ECUDA, "cluster launch failed: %s", cudaGetErrorString(e));
  if (g_prof) {
    cudaEventRecord(g_ev1, stream);
    g_ev_pending = true;
  }
  ++g_launches;
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(FFS_ECUDA, "CUDA error: %s", cudaGetErrorString(e));
  g_err[0] = 0;
  return FFS_OK;
}

// ------------------------------------------------------------------ lockstep-dense path
// Full sampling (N' = N) of real U at large L: per block step, one DMMA GEMM P = U Y for a batch
// of S samples, then one cluster per sample draws on its panel and updates W and Y
// (ffs_dense.cuh, ffs_cluster_kernel<..., STEP = true>).
bool dense_eligible(int64_t L, int64_t N, int64_t Np, int dtype) {
  const char* g = getenv("FFS_NO_DENSE");
  if (g && g[0] == '1') return false;
  // marginals (N' < N) take the same step + batched-GJ kernels with every block contracted gathered
  // (no GEMM): C5 marginal 201 -> 180 ms against the per-sample cluster kernel
  const char* m = getenv("FFS_STEP_MARGINAL");  // development: "0" keeps marginals on the cluster kernel
  const bool marg = !(m && m[0] == '0') && Np < N;
  return (Np == N || marg) && N >= 256 && N % 2 == 0 && cluster_eligible(L, dtype);
}

struct DensePlan {
  ClusterPlan c;
  int64_t S, Sh, ldY;  // batch, half-batch (per stream), Y row stride in scalars of T
  int nstr;            // streams (half-batches) in flight
  bool small_gemm;     // GEMM <16, 4> (co-resident with the GJ kernel) instead of <32, 3>
  bool ozaki;          // Ozaki-emulated GEMM on the INT8 tensor cores instead of the DMMA GEMM
  int Kp;              // GEMM K (f N) padded to the Ozaki K chunk
  size_t ws_oza, ws_ea, ws_ozb, ws_eb;
  size_t ws_perm, ws_y, ws_p, ws_w, ws_ch, ws_row, ws_ut, total, y_half, p_half;
  int k_gather;        // blocks with k0 < k_gather contract the gathered columns in the step kernel
};

// GJ tile: real 128 columns (two per thread, 16-byte W accesses), complex 64
template <typename T> constexpr int gj_tj() { return sizeof(T) == 8 ? 128 : 64; }
template <typename T>
const void* dense_gj_fn() { return reinterpret_cast<const void*>(&ffsk::ffs_dense_gj_kernel<T, 8, gj_tj<T>()>); }
template <typename T>
size_t dense_gj_bytes(int k0) { return ffsk::dense_gj_smem<T, 8, gj_tj<T>()>(k0); }

int make_dense_plan(int64_t L, int64_t N, int64_t Np, int dtype, int64_t M, DensePlan& d) {
  const bool cx = dtype == FFS_C128;
  int rc = make_cluster_plan(L, N, Np, dtype, M, d.c);
  if (rc != FFS_OK) return rc;
  d.c.fn = cx ? ffsk::cluster_step_kernel_ptr<cplx, 2, 8, 512>() : ffsk::cluster_step_kernel_ptr<double, 4, 8, 512>();
  d.c.R = cx ? 2 : 4;
  d.c.B = 8;
  d.c.Lc = 512 * d.c.R;
  d.c.CS = std::max<int>(2, (int)((L + d.c.Lc - 1) / d.c.Lc));
  if (d.c.CS > 8) d.c.CS = 16;
  d.c.Lpt = d.c.CS * d.c.Lc;
  if (cudaFuncSetAttribute(d.c.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)d.c.smem) != cudaSuccess)
    return fail(FFS_ECUDA, "cudaFuncSetAttribute(step smem) failed");
  if (d.c.CS > 8 && cudaFuncSetAttribute(d.c.fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
    return fail(FFS_ECUDA, "non-portable cluster size not allowed");
  // one stream and the <32, 3> GEMM: two half-batches on two streams with the co-residable
  // <16, 4> GEMM + 128-thread GJ measured no overlap gain (C4 1.570 vs 1.526 s, C5 1.663 vs 1.549 s)
  d.nstr = 1;
  if (const char* e = getenv("FFS_DENSE_STREAMS")) d.nstr = std::max(1, std::min(2, atoi(e)));  // development
  d.small_gemm = false;
  if (const char* e = getenv("FFS_DENSE_GEMM")) d.small_gemm = atoi(e) == 16;  // development
  const void* gf = d.small_gemm ? reinterpret_cast<const void*>(&ffsk::ffs_dgemm_kernel<16, 4>)
                                : reinterpret_cast<const void*>(&ffsk::ffs_dgemm_kernel<32, 3>);
  const size_t gsm = d.small_gemm ? ffsk::gemm_smem<16, 4>() : ffsk::gemm_smem<32, 3>();
  if (cudaFuncSetAttribute(gf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsm) != cudaSuccess)
    return fail(FFS_ECUDA, "cudaFuncSetAttribute(gemm smem) failed");
  // samples per lockstep batch: as many as ~24 GB of per-sample factors W allow (larger batches =
  // larger GEMMs and fewer launches: C4 1.188 s at 1024, 1.161 s at 4096), at least 1024, at most
  // 8192 (marginals have no GEMM operands)
  const double wbytes = (double)Np * (double)Np * (dtype == FFS_C128 ? 16.0 : 8.0);
  int64_t cap = std::max<int64_t>(1024, std::min<int64_t>(8192, (int64_t)(24e9 / wbytes)));
  if (const char* e = getenv("FFS_DENSE_S")) cap = std::max<int64_t>(1, atoll(e));  // development
  d.S = std::max<int64_t>(1, std::min<int64_t>(M, cap));
  if (d.S < 2) d.nstr = 1;
  d.Sh = (d.S + d.nstr - 1) / d.nstr;
  // ldY in scalars of T; the GEMM's N (2 ldY real columns for complex) is a multiple of 128
  const int64_t q = cx ? ffsk::kGN / 2 : ffsk::kGN;
  d.ldY = (d.Sh * d.c.B + q - 1) / q * q;
  const size_t es = cx ? 16 : 8;
  const bool no_gemm = Np < N;  // marginals: gathered contraction only (the GEMM would be N/N' x wasteful)
  d.y_half = no_gemm ? 0 : align_up((size_t)N * d.ldY * es * (cx ? 2 : 1));  // complex: 2N x 2ldY expansion
  d.p_half = no_gemm ? 0 : align_up((size_t)L * d.ldY * es);
  d.ws_perm = align_up((size_t)std::max<int64_t>(M, 1) * Np * 4);
  d.ws_y = d.nstr * d.y_half;
  d.ws_p = d.nstr * d.p_half;
  d.ws_w = align_up((size_t)d.nstr * d.Sh * Np * Np * es);
  d.ws_ch = align_up((size_t)d.nstr * d.Sh * (d.c.Lpt / 32) * 4);
  d.ws_row = align_up((size_t)d.nstr * d.Sh * (d.c.B * d.c.B + d.c.B) * es);
  // GEMM: Ozaki-style FP64 emulation on the INT8 tensor cores by default (2x the DMMA GEMM at the
  // C5 block shape); FFS_DENSE_GEMM=dmma selects the DMMA GEMM
  const char* gsel = getenv("FFS_DENSE_GEMM");
  d.ozaki = !(gsel && (strcmp(gsel, "dmma") == 0 || atoi(gsel) > 0)) && d.nstr == 1 && !no_gemm;
  // hybrid: while k0 is small the gathered contraction (L k0 B per sample, from the transposed U)
  // costs less than the GEMM's full-N one (L N B); crossover measured on C4/C5:
  // Ozaki GEMM: C5 0.15-0.2 -> 0.97 s (1.01 s at 0), C4 0.35-0.4 -> 0.94 s (0.99 s at 0.6);
  // DMMA GEMM: C5 0.3 -> 1.35 s, C4 0.6 -> 1.19 s. Complex contractions do 2x the flops per
  // gathered byte, so gathering pays longer.
  double theta = d.ozaki ? (cx ? 0.35 : 0.15) : (cx ? 0.6 : 0.3);
  if (const char* e = getenv("FFS_DENSE_THETA")) theta = atof(e);  // development
  d.k_gather = no_gemm ? (int)Np : (int)(theta * (double)Np);
  d.ws_ut = d.k_gather > 0 ? align_up((size_t)N * d.c.Lpt * es) : 0;
  const int64_t fK = (cx ? 2 : 1) * N;
  d.Kp = (int)((fK + ffsk::kOzBK - 1) / ffsk::kOzBK * ffsk::kOzBK);
  const int64_t ncolsY = (cx ? 2 : 1) * d.ldY;
  d.ws_oza = d.ozaki ? align_up((size_t)ffsk::kOzS * L * d.Kp) : 0;
  d.ws_ea = d.ozaki ? align_up((size_t)L * 4) : 0;
  d.ws_ozb = d.ozaki ? align_up((size_t)ffsk::kOzS * ncolsY * d.Kp) : 0;
  d.ws_eb = d.ozaki ? align_up((size_t)ncolsY * 4) : 0;
  if (d.ozaki && cudaFuncSetAttribute(reinterpret_cast<const void*>(&ffsk::ffs_ozaki_gemm_kernel),
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ffsk::kOzSmem) != cudaSuccess)
    return fail(FFS_ECUDA, "cudaFuncSetAttribute(ozaki smem) failed");
  d.total = d.ws_perm + d.ws_y + d.ws_p + d.ws_w + d.ws_ch + d.ws_row + d.ws_ut + d.ws_oza + d.ws_ea + d.ws_ozb + d.ws_eb;
  const size_t gjs = cx ? dense_gj_bytes<cplx>((int)Np) : dense_gj_bytes<double>((int)Np);
  if (gjs > kMaxSmem) return fail(FFS_EINVAL, "dense path: N'=%lld too large for the GJ tile", (long long)Np);
  const void* gjf = cx ? dense_gj_fn<cplx>() : dense_gj_fn<double>();
  if (cudaFuncSetAttribute(gjf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gjs) != cudaSuccess)
    return fail(FFS_ECUDA, "cudaFuncSetAttribute(gj smem) failed");
  return FFS_OK;
}

// 3-D tensor map [kOzS][rows][Kp] of int8 slices, box {kOzBK, box_rows, 1}, 64-byte swizzle
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int oz_tensor_map(CUtensorMap* m, const int8_t* base, int64_t rows, int Kp, int box_rows) {
  // resolved once (thread-safe function-local static)
  static const EncodeTiledFn enc = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess) fn = nullptr;
    return reinterpret_cast<EncodeTiledFn>(fn);
  }();
  if (!enc) return fail(FFS_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[3] = {(cuuint64_t)Kp, (cuuint64_t)rows, (cuuint64_t)ffsk::kOzS};
  const cuuint64_t strides[2] = {(cuuint64_t)Kp, (cuuint64_t)Kp * (cuuint64_t)rows};
  const cuuint32_t box[3] = {(cuuint32_t)ffsk::kOzBK, (cuuint32_t)box_rows, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  if (enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return fail(FFS_ECUDA, "cuTensorMapEncodeTiled failed");
  return FFS_OK;
}

// a second stream (and fork/join events) per host thread for the 2-stream dense schedule
thread_local cudaStream_t g_dense_s1 = nullptr;
thread_local cudaEvent_t g_dense_fork = nullptr, g_dense_join = nullptr;

int launch_dense(const void* U, int64_t L, int64_t N, int dtype, int64_t M, int64_t Np, const double* uniforms,
                 int32_t* positions, int32_t* flags, void* ws, size_t ws_bytes, cudaStream_t stream, int64_t S,
                 double* trace) {
  const bool cx = dtype == FFS_C128;
  DensePlan d;
  int rc = make_dense_plan(L, N, Np, dtype, M, d);
  if (rc != FFS_OK) return rc;
  if (!ws || ws_bytes < d.total) return fail(FFS_EINVAL, "workspace %zu bytes < required %zu", ws_bytes, d.total);
  if (((uintptr_t)ws & (kAlign - 1)) != 0) return fail(FFS_EINVAL, "workspace not 256-byte aligned");
  const size_t es = cx ? 16 : 8;
  const int B = d.c.B;
  char* w = static_cast<char*>(ws);
  int32_t* perm = reinterpret_cast<int32_t*>(w);
  char* Yb = w + d.ws_perm;
  char* Pb = Yb + d.ws_y;
  char* Wb = Pb + d.ws_p;
  uint32_t* ch = reinterpret_cast<uint32_t*>(Wb + d.ws_w);
  char* rowb = Wb + d.ws_w + d.ws_ch;
  double* Ut = reinterpret_cast<double*>(rowb + d.ws_row);
  char* ozb0 = rowb + d.ws_row + d.ws_ut;
  int8_t* oza = reinterpret_cast<int8_t*>(ozb0);
  int* oz_ea = reinterpret_cast<int*>(ozb0 + d.ws_oza);
  int8_t* ozb = reinterpret_cast<int8_t*>(ozb0 + d.ws_oza + d.ws_ea);
  int* oz_eb = reinterpret_cast<int*>(ozb0 + d.ws_oza + d.ws_ea + d.ws_ozb);
  CUtensorMap oz_ta, oz_tb;
  const int64_t oz_ncols = (cx ? 2 : 1) * d.ldY;
  if (d.ozaki) {
    if (oz_tensor_map(&oz_ta, oza, L, d.Kp, ffsk::kOzBM) != FFS_OK) return FFS_ECUDA;
    if (oz_tensor_map(&oz_tb, ozb, oz_ncols, d.Kp, ffsk::kOzBN) != FFS_OK) return FFS_ECUDA;
    // A = U (real L x 2N view for complex): split once per call
    const int64_t fK = (cx ? 2 : 1) * N;
    ffsk::ffs_ozaki_split_rows_kernel<<<(unsigned)((L + 7) / 8), 256, 0, stream>>>(
        static_cast<const double*>(U), (int)L, (int)fK, fK, oza, d.Kp, oz_ea);
    ++g_launches;
  }
  if (d.k_gather > 0) {
    dim3 tb(32, 8), tg((unsigned)((d.c.Lpt + 31) / 32), (unsigned)((N + 31) / 32));
    if (cx) ffsk::transpose_pad_kernel<cplx><<<tg, tb, 0, stream>>>(static_cast<const double*>(U), Ut, (int)L, (int)N, d.c.Lpt);
    else ffsk::transpose_pad_kernel<double><<<tg, tb, 0, stream>>>(static_cast<const double*>(U), Ut, (int)L, (int)N, d.c.Lpt);
    ++g_launches;
  }
  cudaStream_t st[2] = {stream, stream};
  if (d.nstr > 1) {
    if (!g_dense_s1) {
      if (cudaStreamCreateWithFlags(&g_dense_s1, cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&g_dense_fork, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&g_dense_join, cudaEventDisableTiming) != cudaSuccess)
        return fail(FFS_ECUDA, "dense path: stream/event creation failed");
    }
    st[1] = g_dense_s1;
  }
  if (g_prof) {
    if (!g_ev0) {
      cudaEventCreate(&g_ev0);
      cudaEventCreate(&g_ev1);
    }
    cudaEventRecord(g_ev0, stream);
  }
  {
    const int tpb = (int)std::max<int64_t>(1, std::min<int64_t>(128, 40960 / (4 * N)));
    const int64_t pgrid = (M + tpb - 1) / tpb;
    ffsk::ffs_permute_kernel<<<(unsigned)pgrid, tpb, (size_t)tpb * N * 4, stream>>>(uniforms, perm, M, (int)N,
                                                                                       (int)Np);
    ++g_launches;
  }
  if (d.nstr > 1) {
    cudaEventRecord(g_dense_fork, stream);
    cudaStreamWaitEvent(st[1], g_dense_fork, 0);
  }
  const int64_t f = cx ? 2 : 1;
  const void* gjf = cx ? dense_gj_fn<cplx>() : dense_gj_fn<double>();
  const int gjt = cx ? gj_tj<cplx>() : gj_tj<double>();
  const size_t rstride = (size_t)(B * B + B) * es;
  for (int64_t base = 0; base < M; base += d.S) {
    const int64_t Sb = std::min<int64_t>(d.S, M - base);
    ffsk::ClusterParams p[2] = {};
    ffsk::DgemmParams gp[2] = {};
    ffsk::DenseGjParams q[2] = {};
    int64_t nh[2] = {0, 0};
    for (int h = 0; h < d.nstr; ++h) {
      const int64_t b0 = std::min<int64_t>(Sb, h * d.Sh);
      nh[h] = std::min<int64_t>(Sb, b0 + d.Sh) - b0;
      if (nh[h] <= 0) continue;
      double* Y = reinterpret_cast<double*>(Yb + h * d.y_half);
      double* Pd = reinterpret_cast<double*>(Pb + h * d.p_half);
      double* Wd = reinterpret_cast<double*>(Wb + (size_t)h * d.Sh * Np * Np * es);
      uint32_t* chh = ch + (size_t)h * d.Sh * (d.c.Lpt / 32);
      double* rowg = reinterpret_cast<double*>(rowb + (size_t)h * d.Sh * rstride);
      if (d.y_half) cudaMemsetAsync(Y, 0, d.y_half, st[h]);
      cudaMemsetAsync(chh, 0, (size_t)nh[h] * (d.c.Lpt / 32) * 4, st[h]);
      if (flags) cudaMemsetAsync(flags + base + b0, 0, (size_t)nh[h] * 4, st[h]);
      const unsigned yg = (unsigned)((nh[h] * B + 255) / 256);
      if (!d.y_half) Y = nullptr;
      else if (cx) ffsk::ffs_dense_y0_kernel<cplx, 8><<<yg, 256, 0, st[h]>>>(perm, Y, d.ldY, base + b0, (int)nh[h], (int)Np);
      else ffsk::ffs_dense_y0_kernel<double, 8><<<yg, 256, 0, st[h]>>>(perm, Y, d.ldY, base + b0, (int)nh[h], (int)Np);
      if (Y) ++g_launches;
      ffsk::ClusterParams& c = p[h];
      c.U = static_cast<const double*>(U);
      c.Ut = Ut;
      c.L = (int)L;
      c.N = (int)N;
      c.Np = (int)Np;
      c.Lc = d.c.Lc;
      c.Lpt = d.c.Lpt;
      c.M = M;
      c.uniforms = uniforms;
      c.positions = positions;
      c.flags = flags;
      c.wfull = Wd;
      c.S = S > 0 ? std::min<int64_t>(S, M) : 0;
      c.trace = S > 0 ? trace : nullptr;
      c.timing = g_timing;  // development (ffs_dev_timing); null unless enabled
      c.Pd = Pd;
      c.ldY = d.ldY;
      c.rowg = rowg;
      c.permg = perm;
      c.chosen_g = chh;
      c.base = base + b0;
      c.Sb = (int)nh[h];
      // complex: the real GEMM of U viewed as L x 2N with the real 2N x 2ldY expansion of Y
      gp[h].A = static_cast<const double*>(U);
      gp[h].B = Y;
      gp[h].C = Pd;
      gp[h].lda = f * N;
      gp[h].ldb = f * d.ldY;
      gp[h].ldc = f * d.ldY;
      gp[h].M = (int)L;
      gp[h].N = (int)(f * d.ldY);
      gp[h].K = (int)(f * N);
      gp[h].panel = (int)(f * B);  // P in per-sample [L][B] panels (contiguous reads in the step kernel)
      q[h].U = static_cast<const double*>(U);
      q[h].perm = perm;
      q[h].positions = positions;
      q[h].rowg = rowg;
      q[h].W = Wd;
      q[h].Y = Y;
      q[h].ldY = d.ldY;
      q[h].N = (int)N;
      q[h].Np = (int)Np;
      q[h].base = base + b0;
    }
    const dim3 ggrid((unsigned)(f * d.ldY / ffsk::kGN), (unsigned)((L + ffsk::kGM - 1) / ffsk::kGM));
    for (int k0 = 0; k0 < Np; k0 += B) {
      for (int h = 0; h < d.nstr; ++h) {
        if (nh[h] <= 0) continue;
        p[h].gather = k0 < d.k_gather ? 1 : 0;
        if (p[h].gather) {
          // no GEMM: the step kernel contracts the gathered columns itself
        } else if (d.ozaki) {
          ffsk::ffs_ozaki_split_cols_kernel<<<(unsigned)(oz_ncols / 32), 256, 0, st[h]>>>(
              gp[h].B, (int)gp[h].K, (int)oz_ncols, gp[h].ldb, ozb, d.Kp, oz_eb);
          ffsk::OzakiParams op{};
          op.ea = oz_ea;
          op.eb = oz_eb;
          op.C = gp[h].C;
          op.M = (int)L;
          op.N = (int)oz_ncols;
          op.K = d.Kp;
          op.panel = gp[h].panel;
          const dim3 og((unsigned)(oz_ncols / ffsk::kOzBN), (unsigned)((L + ffsk::kOzBM - 1) / ffsk::kOzBM));
          ffsk::ffs_ozaki_gemm_kernel<<<og, ffsk::kOzThreads, ffsk::kOzSmem, st[h]>>>(oz_ta, oz_tb, op);
          g_launches += 1;
        } else if (d.small_gemm)
          ffsk::ffs_dgemm_kernel<16, 4><<<ggrid, ffsk::kGThreads, ffsk::gemm_smem<16, 4>(), st[h]>>>(gp[h]);
        else
          ffsk::ffs_dgemm_kernel<32, 3><<<ggrid, ffsk::kGThreads, ffsk::gemm_smem<32, 3>(), st[h]>>>(gp[h]);
        if (!p[h].gather) ++g_launches;
        p[h].k0 = k0;
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = d.c.CS;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.blockDim = dim3(d.c.threads);
        cfg.gridDim = dim3((unsigned)(nh[h] * d.c.CS));
        cfg.dynamicSmemBytes = d.c.smem;
        cfg.stream = st[h];
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        void* args[] = {&p[h]};
        cudaError_t e = cudaLaunchKernelExC(&cfg, d.c.fn, args);
        if (e != cudaSuccess) return fail(FFS_ECUDA, "step launch failed: %s", cudaGetErrorString(e));
        ++g_launches;
        if (k0 + B < Np) {
          q[h].k0 = k0;
          const int nc = (int)Np - k0 - B;
          const dim3 jg((unsigned)((nc + gjt - 1) / gjt), (unsigned)nh[h]);
          const size_t gsm = cx ? dense_gj_bytes<cplx>(k0) : dense_gj_bytes<double>(k0);
          void* qargs[] = {&q[h]};
          e = cudaLaunchKernel(gjf, jg, dim3(256), qargs, gsm, st[h]);
          if (e != cudaSuccess) return fail(FFS_ECUDA, "gj launch failed: %s", cudaGetErrorString(e));
          ++g_launches;
        }
      }
    }
  }
  if (d.nstr > 1) {
    cudaEventRecord(g_dense_join, st[1]);
    cudaStreamWaitEvent(stream, g_dense_join, 0);
  }
  if (g_prof) {
    cudaEventRecord(g_ev1, stream);
    g_ev_pending = true;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(FFS_ECUDA, "CUDA error: %s", cudaGetErrorString(e));
  g_err[0] = 0;
  return FFS_OK;
}

bool use_warp_path(int64_t L, int64_t N, int64_t Np, int dtype) {
  const char* g = getenv("FFS_FORCE_GENERIC");
  if (g && g[0] == '1') return false;
  return warp_eligible(L, N, Np, dtype);
}

int launch(const void* U, int64_t L, int64_t N, int dtype, int64_t M, int64_t Np, const double* uniforms,
           int32_t* positions, int32_t* flags, void* ws, size_t ws_bytes, cudaStream_t stream, int64_t S,
           double* trace) {
  g_launches = 0;
  if (M == 0) return FFS_OK;
  if (L < 1 || N < 1 || N > L || Np < 1 || Np > N || L > INT32_MAX || M < 0)
    return fail(FFS_EINVAL, "invalid shape L=%lld N=%lld N'=%lld M=%lld", (long long)L, (long long)N,
                (long long)Np, (long long)M);
  if (dtype != FFS_F64 && dtype != FFS_C128) return fail(FFS_EINVAL, "unknown dtype %d", dtype);
  if (!U || !uniforms || !positions) return fail(FFS_EINVAL, "null U/uniforms/positions with M=%lld", (long long)M);
  if (S > 0 && !trace) return fail(FFS_EINVAL, "null trace buffer with S=%lld", (long long)S);
  if (use_warp_path(L, N, Np, dtype))
    return launch_warp(U, L, N, M, Np, uniforms, positions, flags, ws, ws_bytes, stream, S, trace);
  if (dense_eligible(L, N, Np, dtype))
    return launch_dense(U, L, N, dtype, M, Np, uniforms, positions, flags, ws, ws_bytes, stream, S, trace);
  if (cluster_eligible(L, dtype))
    return launch_cluster(U, L, N, dtype, M, Np, uniforms, positions, flags, ws, ws_bytes, stream, S, trace);
  Plan pl;
  int rc = make_plan(L, N, Np, dtype, M, pl);
  if (rc != FFS_OK) return rc;
  if (!U || !uniforms || !positions) return fail(FFS_EINVAL, "null U/uniforms/positions with M=%lld", (long long)M);
  if (S > 0 && !trace) return fail(FFS_EINVAL, "null trace buffer with S=%lld", (long long)S);
  const size_t need = pl.ws_ut + pl.ws_wfull;
  if (need > 0 && (!ws || ws_bytes < need))
    return fail(FFS_EINVAL, "workspace %zu bytes < required %zu", ws_bytes, need);
  if (((uintptr_t)ws & (kAlign - 1)) != 0) return fail(FFS_EINVAL, "workspace not 256-byte aligned");
  char* w = static_cast<char*>(ws);
  ffsk::Params p{};
  if (const char* dbg = getenv("FFS_DEBUG_SKIP")) p.dbg = atoi(dbg);  // development only
  p.U = static_cast<const double*>(U);
  p.Ut = pl.v.usmem ? nullptr : reinterpret_cast<const double*>(w);
  p.L = (int)L;
  p.N = (int)N;
  p.Np = (int)Np;
  p.Lp = pl.Lp;
  p.ut_stride = pl.ut_stride;
  p.M = M;
  p.uniforms = uniforms;
  p.positions = positions;
  p.flags = flags;
  p.wfull = reinterpret_cast<double*>(w + pl.ws_ut);
  p.S = S > 0 ? std::min<int64_t>(S, M) : 0;
  p.trace = S > 0 ? trace : nullptr;
  p.owner_smem = pl.owner_smem;
  p.ushared_smem = pl.ushared_smem;
  if (!pl.v.usmem) {
    dim3 tb(32, 8), tg((unsigned)((pl.Lp + 31) / 32), (unsigned)((N + 31) / 32));
    if (dtype == FFS_C128)
      ffsk::transpose_pad_kernel<cplx><<<tg, tb, 0, stream>>>(p.U, const_cast<double*>(p.Ut), (int)L, (int)N, pl.Lp);
    else
      ffsk::transpose_pad_kernel<double><<<tg, tb, 0, stream>>>(p.U, const_cast<double*>(p.Ut), (int)L, (int)N, pl.Lp);
    ++g_launches;
  }
  void* args[] = {&p};
  cudaError_t e = launch_timed(pl.v.fn, dim3(pl.grid), dim3(pl.threads), args, pl.smem, stream);
  if (e != cudaSuccess) return fail(FFS_ECUDA, "launch failed: %s", cudaGetErrorString(e));
  ++g_launches;
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(FFS_ECUDA, "CUDA error: %s", cudaGetErrorString(e));
  g_err[0] = 0;
  return FFS_OK;
}

}  // namespace

extern "C" {

size_t ffs_workspace_bytes(int64_t L, int64_t N, int64_t Nprime, int dtype, int64_t M) {
  if (L >= 1 && N >= 1 && N <= L && Nprime >= 1 && Nprime <= N && use_warp_path(L, N, Nprime, dtype)) {
    WarpPlan w;
    if (make_warp_plan(L, N, Nprime, std::max<int64_t>(M, 1), w) != FFS_OK) return 0;
    return w.ws_perm + w.ws_w;
  }
  if (L >= 1 && N >= 1 && N <= L && Nprime >= 1 && Nprime <= N && dense_eligible(L, N, Nprime, dtype)) {
    DensePlan d;
    if (make_dense_plan(L, N, Nprime, dtype, std::max<int64_t>(M, 1), d) != FFS_OK) return 0;
    return d.total;
  }
  if (L >= 1 && N >= 1 && N <= L && Nprime >= 1 && Nprime <= N && cluster_eligible(L, dtype)) {
    ClusterPlan c;
    if (make_cluster_plan(L, N, Nprime, dtype, std::max<int64_t>(M, 1), c) != FFS_OK) return 0;
    return c.ws_ut + c.ws_w;
  }
  Plan pl;
  if (make_plan(L, N, Nprime, dtype, std::max<int64_t>(M, 1), pl) != FFS_OK) return 0;
  return pl.ws_ut + pl.ws_wfull;
}

int ffs_sample(const void* U, int64_t L, int64_t N, int dtype, int64_t M, const double* uniforms,
               int32_t* positions, int32_t* sample_flags, void* workspace, size_t ws_bytes, void* stream) {
  return launch(U, L, N, dtype, M, N, uniforms, positions, sample_flags, workspace, ws_bytes,
                static_cast<cudaStream_t>(stream), 0, nullptr);
}

int ffs_sample_marginal(const void* U, int64_t L, int64_t N, int dtype, int64_t M, int64_t Nprime,
                        const double* uniforms, int32_t* positions, int32_t* sample_flags, void* workspace,
                        size_t ws_bytes, void* stream) {
  return launch(U, L, N, dtype, M, Nprime, uniforms, positions, sample_flags, workspace, ws_bytes,
                static_cast<cudaStream_t>(stream), 0, nullptr);
}

int ffs_debug_trace(const void* U, int64_t L, int64_t N, int dtype, int64_t M, int64_t Nprime,
                    const double* uniforms, int32_t* positions, int32_t* sample_flags, void* workspace,
                    size_t ws_bytes, void* stream, int64_t S, double* weights) {
  return launch(U, L, N, dtype, M, Nprime, uniforms, positions, sample_flags, workspace, ws_bytes,
                static_cast<cudaStream_t>(stream), S, weights);
}

// ---------------------------------------------------------------- host-buffer path
// Device layout inside the caller's workspace: [U | uniforms chunk x2 | positions chunk x2 |
// flags chunk x2 | sampling workspace]. Chunks alternate between two buffers so the copies of
// chunk c+1 overlap the kernel of chunk c on the caller's stream (copies and kernels of one
// stream serialise; overlap comes from a second stream created lazily per thread).
namespace {
struct HostLayout {
  size_t u, uni[2], pos[2], flg[2], ws, total;
  int64_t chunk;
};
int64_t host_chunk(int64_t M) { return std::max<int64_t>(1, std::min<int64_t>(M, M > 32768 ? 16384 : M)); }
bool host_layout(int64_t L, int64_t N, int64_t Np, int dtype, int64_t M, HostLayout& h) {
  const size_t es = dtype == FFS_C128 ? 16 : 8;
  h.chunk = host_chunk(M);
  size_t o = 0;
  h.u = o; o = align_up(o + (size_t)L * N * es);
  for (int b = 0; b < 2; ++b) { h.uni[b] = o; o = align_up(o + (size_t)h.chunk * 2 * Np * 8); }
  for (int b = 0; b < 2; ++b) { h.pos[b] = o; o = align_up(o + (size_t)h.chunk * Np * 4); }
  for (int b = 0; b < 2; ++b) { h.flg[b] = o; o = align_up(o + (size_t)h.chunk * 4); }
  h.ws = o;
  const size_t need = ffs_workspace_bytes(L, N, Np, dtype, h.chunk);
  if (need == 0) return false;
  o += need;
  h.total = o;
  return true;
}
}  // namespace

size_t ffs_host_workspace_bytes(int64_t L, int64_t N, int64_t Nprime, int dtype, int64_t M) {
  HostLayout h;
  if (!host_layout(L, N, Nprime, dtype, std::max<int64_t>(M, 1), h)) return 0;
  return h.total;
}

// Three-stage pipeline over sample chunks, double-buffered in the workspace: copy-in stream
// (U once, then uniforms of chunk c) -> caller's stream (sampling of chunk c) -> copy-out stream
// (positions/flags of chunk c). Chunk c+1's upload and chunk c-1's download overlap chunk c's
// kernels. Streams/events are created once per host thread (no device memory is allocated).
namespace {
struct HostPipe {
  cudaStream_t ci = nullptr, co = nullptr;
  cudaEvent_t entry, in_ready[2], done[2], out_done[2];
  bool ok = false;
  bool init() {
    if (ok) return true;
    if (cudaStreamCreateWithFlags(&ci, cudaStreamNonBlocking) != cudaSuccess) return false;
    if (cudaStreamCreateWithFlags(&co, cudaStreamNonBlocking) != cudaSuccess) return false;
    if (cudaEventCreateWithFlags(&entry, cudaEventDisableTiming) != cudaSuccess) return false;
    for (int b = 0; b < 2; ++b) {
      if (cudaEventCreateWithFlags(&in_ready[b], cudaEventDisableTiming) != cudaSuccess) return false;
      if (cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming) != cudaSuccess) return false;
      if (cudaEventCreateWithFlags(&out_done[b], cudaEventDisableTiming) != cudaSuccess) return false;
    }
    ok = true;
    return true;
  }
};
thread_local HostPipe g_pipe;
}  // namespace

int ffs_sample_host(const void* U, int64_t L, int64_t N, int dtype, int64_t M, int64_t Nprime,
                    const double* uniforms, int32_t* positions, int32_t* sample_flags, void* workspace,
                    size_t ws_bytes, void* stream) {
  if (M == 0) return FFS_OK;
  HostLayout h;
  if (!host_layout(L, N, Nprime, dtype, M, h)) return FFS_EINVAL;
  if (!U || !uniforms || !positions || !workspace || ws_bytes < h.total)
    return fail(FFS_EINVAL, "host path: null pointer or workspace %zu < %zu", ws_bytes, h.total);
  if (!g_pipe.init()) return fail(FFS_ECUDA, "host path: stream/event creation failed");
  cudaStream_t s0 = static_cast<cudaStream_t>(stream);
  HostPipe& hp = g_pipe;
  char* w = static_cast<char*>(workspace);
  const size_t es = dtype == FFS_C128 ? 16 : 8;
  const int64_t Np = Nprime;
  int launches = 0;
  cudaError_t e = cudaSuccess;
#define FFS_CK(x, what) do { e = (x); if (e != cudaSuccess) return fail(FFS_ECUDA, "%s: %s", what, cudaGetErrorString(e)); } while (0)
  FFS_CK(cudaEventRecord(hp.entry, s0), "record");          // prior work on the caller's stream
  FFS_CK(cudaStreamWaitEvent(hp.ci, hp.entry, 0), "wait");
  FFS_CK(cudaMemcpyAsync(w + h.u, U, (size_t)L * N * es, cudaMemcpyHostToDevice, hp.ci), "H2D U");
  const int64_t nchunks = (M + h.chunk - 1) / h.chunk;
  for (int64_t c = 0; c < nchunks; ++c) {
    const int b = (int)(c & 1);
    const int64_t c0 = c * h.chunk;
    const int64_t mc = std::min<int64_t>(h.chunk, M - c0);
    if (c >= 2) FFS_CK(cudaStreamWaitEvent(hp.ci, hp.done[b], 0), "wait");  // uniforms[b] consumed
    FFS_CK(cudaMemcpyAsync(w + h.uni[b], uniforms + c0 * 2 * Np, (size_t)mc * 2 * Np * 8, cudaMemcpyHostToDevice,
                           hp.ci), "H2D uniforms");
    FFS_CK(cudaEventRecord(hp.in_ready[b], hp.ci), "record");
    FFS_CK(cudaStreamWaitEvent(s0, hp.in_ready[b], 0), "wait");
    if (c >= 2) FFS_CK(cudaStreamWaitEvent(s0, hp.out_done[b], 0), "wait");  // positions[b] drained
    int rc = launch(w + h.u, L, N, dtype, mc, Np, reinterpret_cast<const double*>(w + h.uni[b]),
                    reinterpret_cast<int32_t*>(w + h.pos[b]), reinterpret_cast<int32_t*>(w + h.flg[b]), w + h.ws,
                    h.total - h.ws, s0, 0, nullptr);
    if (rc != FFS_OK) return rc;
    launches += g_launches;
    FFS_CK(cudaEventRecord(hp.done[b], s0), "record");
    FFS_CK(cudaStreamWaitEvent(hp.co, hp.done[b], 0), "wait");
    FFS_CK(cudaMemcpyAsync(positions + c0 * Np, w + h.pos[b], (size_t)mc * Np * 4, cudaMemcpyDeviceToHost, hp.co),
           "D2H positions");
    if (sample_flags)
      FFS_CK(cudaMemcpyAsync(sample_flags + c0, w + h.flg[b], (size_t)mc * 4, cudaMemcpyDeviceToHost, hp.co),
             "D2H flags");
    FFS_CK(cudaEventRecord(hp.out_done[b], hp.co), "record");
  }
  FFS_CK(cudaStreamSynchronize(hp.co), "host path sync");
  FFS_CK(cudaStreamSynchronize(s0), "host path sync");
#undef FFS_CK
  g_launches = launches;
  return FFS_OK;
}

int ffs_last_launch_count(void) { return g_launches; }

// development only (not in ffs.h): per-phase clock64 sums of the segmented warp kernel
int ffs_dev_timing(unsigned long long* host8, int reset) {
  if (!g_timing) {
    if (cudaMalloc(&g_timing, 8 * sizeof(unsigned long long)) != cudaSuccess) return FFS_ECUDA;
    cudaMemset(g_timing, 0, 8 * sizeof(unsigned long long));
  }
  if (host8) cudaMemcpy(host8, g_timing, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  if (reset) cudaMemset(g_timing, 0, 8 * sizeof(unsigned long long));
  return FFS_OK;
}

int ffs_profile_enable(int on) {
  g_prof = on != 0;
  g_ev_pending = false;
  return FFS_OK;
}

float ffs_last_kernel_ms(void) {
  if (!g_ev_pending) return -1.0f;
  float ms = -1.0f;
  if (cudaEventSynchronize(g_ev1) != cudaSuccess) return -1.0f;
  if (cudaEventElapsedTime(&ms, g_ev0, g_ev1) != cudaSuccess) return -1.0f;
  return ms;
}

const char* ffs_last_error(void) { return g_err; }

}  // extern "C"
