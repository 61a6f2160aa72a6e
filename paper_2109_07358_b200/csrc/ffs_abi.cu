// C ABI of libffs.so (declarations and contracts: include/ffs.h).
// Argument validation, plan selection (cached per shape), workspace carving, the CUDA-graph
// driver of the block-step paths, and the host-buffer path. No torch types and no hidden device
// allocations; every step of the method runs in the kernels of ffs_*.cuh.
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <map>
#include <mutex>
#include <set>
#include <tuple>
#include <utility>
#include <vector>

#include "ffs.h"
#include "ffs_host.h"
#include "ffs_kernel.cuh"
#include "ffs_warp_kernel.cuh"
#include "ffs_cluster_kernel.cuh"
#include "ffs_dense.cuh"
#include "ffs_gram.cuh"
#include "ffs_kmarg.cuh"
#include "ffs_kmarg_c.cuh"
#include "ffs_lens.cuh"
#include "ffs_observe.cuh"
#include "ffs_metro.cuh"
#include "ffs_hkpv.cuh"
#include "ffs_kptr.h"

// ====================================================================== shared host helpers
namespace ffsh {
namespace {
thread_local char g_err[512] = "";
thread_local int g_launches = 0;
thread_local bool g_prof = false;
thread_local cudaEvent_t g_ev0 = nullptr, g_ev1 = nullptr;
thread_local bool g_ev_pending = false;

constexpr int kNumOpts = 16;
// defaults of include/ffs.h ffs_option
double default_option(int o) {
  switch (o) {
    case FFS_OPT_DENSE_GEMM: return 8.0;
    case FFS_OPT_DENSE_THETA: return -1.0;
    case FFS_OPT_DENSE_BATCH: return 0.0;
    case FFS_OPT_BLOCK_STEP: return 1.0;
    case FFS_OPT_LARGE_L_MARGINAL: return 1.0;
    case FFS_OPT_CLUSTER: return 1.0;
    case FFS_OPT_GRAPH: return 1.0;
    case FFS_OPT_FORCE_GENERIC: return 0.0;
    case FFS_OPT_GEMM_2SM: return 1.0;
    case FFS_OPT_GRAM_DRAW: return 1.0;
    case FFS_OPT_GRAM_KAPPA: return 1e4;
    case FFS_OPT_DENSE_MIN_L: return 2048.0;
    case FFS_OPT_DENSE_MIN_N: return 256.0;
    case FFS_OPT_TILE_GRAM: return 1.0;
    case FFS_OPT_GJ_PAIR: return 1.0;
    default: return 0.0;
  }
}
struct Options {
  std::atomic<double> v[kNumOpts];
  std::atomic<uint64_t> version{1};
  Options() {
    for (int o = 0; o < kNumOpts; ++o) v[o].store(default_option(o));
  }
};
Options& opts() {
  static Options o;
  return o;
}
std::mutex g_attr_mu;
std::set<std::pair<int, const void*>> g_attr_done;
}  // namespace

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}
void clear_error() { g_err[0] = 0; }
int& launches() { return g_launches; }
double option(int o) { return (o > 0 && o < kNumOpts) ? opts().v[o].load() : 0.0; }
uint64_t options_version() { return opts().version.load(); }

int device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}
int sm_count(int dev) {
  static std::mutex mu;
  static std::map<int, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cache[dev] = sms;
  return sms;
}
int ensure_max_smem(const void* fn) {
  const int dev = device();
  std::lock_guard<std::mutex> lk(g_attr_mu);
  if (g_attr_done.count({dev, fn})) return FFS_OK;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxSmem) != cudaSuccess)
    return fail(FFS_ECUDA, "cudaFuncSetAttribute(MaxDynamicSharedMemorySize) failed");
  g_attr_done.insert({dev, fn});
  return FFS_OK;
}

bool profiling() { return g_prof; }
void prof_begin(cudaStream_t s) {
  if (!g_prof) return;
  if (!g_ev0) {
    cudaEventCreate(&g_ev0);
    cudaEventCreate(&g_ev1);
  }
  cudaEventRecord(g_ev0, s);
}
void prof_end(cudaStream_t s) {
  if (!g_prof) return;
  cudaEventRecord(g_ev1, s);
  g_ev_pending = true;
}
}  // namespace ffsh

using ffsh::align_up;
using ffsh::fail;
using ffsh::kAlign;
using ffsh::kMaxSmem;

namespace {

// ====================================================================== plan cache
// Plans depend on the shape, M, the device and the tuning options; they are made once (with the
// CUDA attribute / occupancy queries) and reused by every later call of the same shape.
using PlanKey = std::tuple<int, int, int64_t, int64_t, int64_t, int64_t, int, uint64_t>;
template <typename P>
struct PlanCache {
  std::mutex mu;
  std::map<PlanKey, P> m;
  template <typename F>
  int get(const PlanKey& k, P& out, F&& make) {
    {
      std::lock_guard<std::mutex> lk(mu);
      auto it = m.find(k);
      if (it != m.end()) {
        out = it->second;
        return FFS_OK;
      }
    }
    int rc = make(out);
    if (rc != FFS_OK) return rc;
    std::lock_guard<std::mutex> lk(mu);
    if (m.size() > 256) m.clear();
    m[k] = out;
    return FFS_OK;
  }
};
PlanKey plan_key(int kind, int64_t L, int64_t N, int64_t Np, int64_t M, int dtype) {
  return PlanKey{ffsh::device(), kind, L, N, Np, M, dtype, ffsh::options_version()};
}

// ------------------------------------------------------------------ generic per-sample kernel
// ffs_sample_kernel<T, WARP, R, B, USMEM>: one warp (small L) or one CTA per sample.
struct Variant {
  bool warp;      // owner = one warp (true) or one CTA (false)
  int R, B;       // rows per thread, panel width
  bool usmem;     // U^T held in shared memory (shared by all owners of a CTA)
  int maxt;       // __launch_bounds__ of the instantiation
  const void* fn; // kernel
};

constexpr int kWarpMaxThreads = 320;

template <typename T, bool WARP, int R, int B, bool USMEM, int MAXT = kWarpMaxThreads>
Variant make_variant() {
  return Variant{WARP, R, B, USMEM, MAXT, ffsk::sample_kernel_ptr<T, WARP, R, B, USMEM, MAXT>()};
}

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

// The largest L each dtype supports on the per-sample kernels: the L x B panel of one sample
// lives in one SM's register file (B = 1 at the limit).
constexpr int64_t kMaxLReal = 16384, kMaxLComplex = 8192;

bool pick_variant(int L, int N, int dtype, Variant& v) {
  const bool c = dtype == FFS_C128;
  const size_t es = c ? 16 : 8;
  // U^T in shared memory if the whole (padded) matrix takes <= 96 KB: one copy per CTA,
  // shared by all warp-owners of that CTA.
  auto fits = [&](int R) { return (size_t)N * (size_t)(32 * R + 2) * es <= 96 * 1024; };
  // Warp owners (L <= 256 real / 128 complex): panel R x B per lane in registers.
  // CTA owners: one sample per CTA; the L x B panel must fit the SM's register file, so B
  // shrinks as L grows.
  if (!c) {
    if (L <= 32)  { v = fits(1) ? make_variant<double, true, 1, 8, true>() : make_variant<double, true, 1, 8, false>(); return true; }
    if (L <= 64)  { v = fits(2) ? make_variant<double, true, 2, 8, true>() : make_variant<double, true, 2, 8, false>(); return true; }
    if (L <= 128) { v = fits(4) ? make_variant<double, true, 4, 8, true>() : make_variant<double, true, 4, 8, false>(); return true; }
    if (L <= 256) { v = fits(8) ? make_variant<double, true, 8, 8, true, 256>() : make_variant<double, true, 8, 8, false, 256>(); return true; }
    if (L <= 1024)  { v = make_variant<double, false, 4, 8, false, 256>(); return true; }
    if (L <= 4096)  { v = make_variant<double, false, 4, 4, false, 1024>(); return true; }
    if (L <= 8192)  { v = make_variant<double, false, 8, 2, false, 1024>(); return true; }
    if (L <= kMaxLReal) { v = make_variant<double, false, 16, 1, false, 1024>(); return true; }
  } else {
    if (L <= 32)  { v = fits(1) ? make_variant<cplx, true, 1, 4, true>() : make_variant<cplx, true, 1, 4, false>(); return true; }
    if (L <= 64)  { v = fits(2) ? make_variant<cplx, true, 2, 4, true>() : make_variant<cplx, true, 2, 4, false>(); return true; }
    if (L <= 128) { v = fits(4) ? make_variant<cplx, true, 4, 4, true>() : make_variant<cplx, true, 4, 4, false>(); return true; }
    if (L <= 1024)  { v = make_variant<cplx, false, 4, 4, false, 256>(); return true; }
    if (L <= 4096)  { v = make_variant<cplx, false, 4, 2, false, 1024>(); return true; }
    if (L <= kMaxLComplex) { v = make_variant<cplx, false, 8, 1, false, 1024>(); return true; }
  }
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

int make_plan_uncached(int64_t L, int64_t N, int64_t Np, int dtype, int64_t M, Plan& pl) {
  if (!pick_variant((int)L, (int)N, dtype, pl.v))
    return fail(FFS_EINVAL, "unsupported L=%lld for dtype %d (max %lld real, %lld complex)", (long long)L, dtype,
                (long long)kMaxLReal, (long long)kMaxLComplex);
  const bool c = dtype == FFS_C128;
  pl.es = c ? 16 : 8;
  const int sms = ffsh::sm_count(ffsh::device());
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, pl.v.fn) != cudaSuccess) return fail(FFS_ECUDA, "cudaFuncGetAttributes failed");
  const int regs = std::max(fa.numRegs, 1);
  pl.owner_smem = owner_bytes(c, pl.v.B, (int)N, (int)Np);
  if (pl.v.warp) {
    pl.G = 32;
    pl.Lp = 32 * pl.v.R;
    pl.ut_stride = pl.Lp + (c ? 1 : 2);  // +16 B per column: spreads column bases over banks
    pl.ushared_smem = pl.v.usmem ? ffsk::align16((size_t)N * pl.ut_stride * pl.es) : 0;
    // warps per CTA: bounded by registers (one CTA per SM when U^T is shared), smem, and 10
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
    if (pl.G > pl.v.maxt) return fail(FFS_EINVAL, "variant needs %d threads > %d", pl.G, pl.v.maxt);
  }
  pl.smem = pl.ushared_smem + (size_t)pl.owners_per_cta * pl.owner_smem;
  if (pl.smem > kMaxSmem) return fail(FFS_EINVAL, "shared memory %zu > %zu (N=%lld)", pl.smem, kMaxSmem, (long long)N);
  if (int rc = ffsh::ensure_max_smem(pl.v.fn)) return rc;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pl.v.fn, pl.threads, pl.smem) != cudaSuccess || per_sm < 1)
    return fail(FFS_EINVAL, "kernel does not fit on an SM (threads=%d smem=%zu regs=%d)", pl.threads, pl.smem, regs);
  const int64_t want = (M + pl.owners_per_cta - 1) / pl.owners_per_cta;
  pl.grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)per_sm * sms));
  pl.ws_ut = pl.v.usmem ? 0 : align_up((size_t)N * pl.Lp * pl.es);
  pl.ws_wfull = align_up((size_t)pl.grid * pl.owners_per_cta * (size_t)Np * Np * pl.es);
  return FFS_OK;
}

PlanCache<Plan> g_plans;
int make_plan(int64_t L, int64_t N, int64_t Np, int dtype, int64_t M, Plan& pl) {
  return g_plans.get(plan_key(0, L, N, Np, M, dtype), pl,
                     [&](Plan& p) { return make_plan_uncached(L, N, Np, dtype, M, p); });
}

// a1 for the paths that take precomputed permutation prefixes: one thread per sample, its
// working permutation of N entries in shared memory (ffs_permute_kernel)
int launch_permute(const double* uniforms, int64_t ustride, int32_t* perm, int64_t M, int64_t N, int64_t Np,
                   cudaStream_t s) {
  const int tpb = (int)std::max<int64_t>(1, std::min<int64_t>(128, 40960 / (4 * N)));
  const size_t smem = (size_t)tpb * N * 4;
  if (smem > kMaxSmem) return fail(FFS_EINVAL, "N=%lld too large for the permutation kernel", (long long)N);
  if (int rc = ffsh::ensure_max_smem(reinterpret_cast<const void*>(&ffsk::ffs_permute_kernel))) return rc;
  const int64_t pgrid = (M + tpb - 1) / tpb;
  ffsk::ffs_permute_kernel<<<(unsigned)pgrid, tpb, smem, s>>>(uniforms, ustride, perm, M, (int)N, (int)Np);
  ++ffsh::launches();
  return FFS_OK;
}

// ------------------------------------------------------------------ fast warp-owner path
// Real U, L <= 256, N' <= kMaxNpWarp, U^T small enough for shared memory: ffs_seg_kernel
// (one CTA per SM, G-lane segments of warps = sample owners) after ffs_permute_kernel.
struct WarpPlan {
  const void* fn;
  int R, B, S, G = 32, maxt, warps, grid, Lp, ut_stride;
  size_t ushared, owner, smem, ws_perm;
};

template <int R, int B, int G, int MAXT>
void warp_fn_seg(WarpPlan& w) {
  w.fn = ffsk::seg_kernel_ptr<R, B, G, MAXT>();
  w.R = R;
  w.B = B;
  w.S = 32 / G;  // samples per warp (one per G-lane segment)
  w.G = G;
  w.maxt = MAXT;
}

bool warp_eligible(int64_t L, int64_t N, int64_t Np, int dtype) {
  if (ffsh::option(FFS_OPT_FORCE_GENERIC) != 0.0) return false;
  if (dtype != FFS_F64 || L > 256 || Np > ffsk::kMaxNpWarp || N > 4096) return false;
  return (size_t)N * (256 + 2) * 8 <= 100 * 1024;  // padded U^T fits shared memory
}

int make_warp_plan_uncached(int64_t L, int64_t N, int64_t Np, int64_t M, WarpPlan& w) {
  // segment width by L (measured: profiles/r01_ncu_summary.md); L <= 16 (C1): 4-lane segments,
  // 8 samples per warp (0.086 ms vs 0.092 ms with 8-lane segments); 256 (C2): one sample per warp,
  // 16 owners/SM at 128 registers (12 when 16 W slices do not fit shared memory)
  const size_t ush = ffsk::align16((size_t)N * (256 + 2) * 8);
  const bool fits16 = ush + 16 * ffsk::WarpLayout((int)Np, 4).total <= kMaxSmem;
  if (L <= 16) warp_fn_seg<4, 4, 4, 512>(w);
  else if (L <= 32) warp_fn_seg<4, 4, 8, 512>(w);
  else if (L <= 64) warp_fn_seg<8, 4, 8, 384>(w);
  else if (L <= 128) warp_fn_seg<8, 4, 16, 384>(w);
  else if (fits16) warp_fn_seg<8, 4, 32, 512>(w);
  else warp_fn_seg<8, 4, 32, 384>(w);
  const int sms = ffsh::sm_count(ffsh::device());
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, w.fn) != cudaSuccess) return fail(FFS_ECUDA, "cudaFuncGetAttributes failed");
  w.Lp = w.G * w.R;
  w.ut_stride = w.Lp + 2;
  w.ushared = ffsk::align16((size_t)N * w.ut_stride * 8);
  w.owner = ffsk::WarpLayout((int)Np, w.B).total;  // per sample; a warp holds S slices
  // registers are allocated per SM sub-partition (4 x 16K); warps are spread round-robin
  const int by_regs = 4 * std::max(1, 16384 / (((std::max(fa.numRegs, 1) * 32 + 255) / 256) * 256));
  int warps = std::min(w.maxt / 32, by_regs);
  while (warps > 1 && w.ushared + (size_t)warps * w.S * w.owner > kMaxSmem) --warps;
  w.warps = warps;
  w.smem = w.ushared + (size_t)warps * w.S * w.owner;
  if (w.smem > kMaxSmem) return fail(FFS_EINVAL, "warp path smem %zu too large", w.smem);
  if (int rc = ffsh::ensure_max_smem(w.fn)) return rc;
  const int64_t ctas = (M + (int64_t)warps * w.S - 1) / ((int64_t)warps * w.S);
  w.grid = (int)std::max<int64_t>(1, std::min<int64_t>(ctas, sms));
  w.ws_perm = align_up((size_t)std::max<int64_t>(M, 1) * Np * 4);
  return FFS_OK;
}

PlanCache<WarpPlan> g_warp_plans;
int make_warp_plan(int64_t L, int64_t N, int64_t Np, int64_t M, WarpPlan& w) {
  return g_warp_plans.get(plan_key(1, L, N, Np, M, FFS_F64), w,
                          [&](WarpPlan& p) { return make_warp_plan_uncached(L, N, Np, M, p); });
}

int launch_warp(const void* U, int64_t L, int64_t N, int64_t M, int64_t Np, const double* uniforms,
                int32_t* positions, int32_t* flags, void* ws, size_t ws_bytes, cudaStream_t stream, int64_t S0, int64_t S,
                double* trace) {
  WarpPlan w;
  int rc = make_warp_plan(L, N, Np, M, w);
  if (rc != FFS_OK) return rc;
  if (!ws || ws_bytes < w.ws_perm)
    return fail(FFS_ENOWS, "workspace %zu bytes < required %zu", ws_bytes, w.ws_perm);
  if (((uintptr_t)ws & (kAlign - 1)) != 0) return fail(FFS_EINVAL, "workspace not 256-byte aligned");
  int32_t* perm = static_cast<int32_t*>(ws);
  if (int rc2 = launch_permute(uniforms, 2 * Np, perm, M, N, Np, stream)) return rc2;
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
  p.S0 = S0;
  p.S = S > 0 ? S : 0;
  p.trace = S > 0 ? trace : nullptr;
  void* args[] = {&p};
  ffsh::prof_begin(stream);
  cudaError_t e = cudaLaunchKernel(w.fn, dim3(w.grid), dim3(32 * w.warps), args, w.smem, stream);
  if (e != cudaSuccess) return fail(FFS_ECUDA, "launch failed: %s", cudaGetErrorString(e));
  ffsh::prof_end(stream);
  ++ffsh::launches();
  return FFS_OK;
}

// ------------------------------------------------------------------ tile-Gram path (small N')
// Real U, N' <= 128, 64 N' <= 3 L: the 32 tile Gram matrices of U once per call, then one warp per
// sample (ffs_kmarg.cuh). Workspace: [perm | U^T | K | Gs slots | C slots].
struct KmPlan {
  const void* fn;
  int Rl, Lpt, grid, warps, G;
  bool c_smem, blocked;
  size_t warp_smem, smem, ws_perm, ws_ut, ws_k, ws_c, total;
};

constexpr int64_t kMaxLTileGram = 262144;
bool kmarg_eligible(int64_t L, int64_t N, int64_t Np, int dtype) {
  if (ffsh::option(FFS_OPT_FORCE_GENERIC) != 0.0 || ffsh::option(FFS_OPT_TILE_GRAM) == 0.0) return false;
  // measured against the panel kernels (tools/shape_time.py, profiles/r02/shape_times.log): below
  // L = 2048 the CTA-owner kernel wins from N' ~ 26 on (L = 1024: N' = 32 3.5 vs 4.2 ms); from L = 2048
  // the tile-Gram path wins up to N' = 64 by 3-5x
  // (N' = 96: L = 4096 20.0 vs 24.3 ms, 8192: 25.8 vs 47.2, 16384: 29.9 vs 52.2; N' = 128 loses at
  // L <= 8192 and wins by 12 % at 16384)
  const int64_t np_max = L <= 1024 ? 24 : L < 2048 ? 32 : L < 4096 ? 64 : ffsk::kKmMaxNp;
  if (dtype == FFS_C128) {  // complex: flat forms only (ffs_kmarg_c.cuh), K is 16 G N^2 bytes; L as for real U
    const int owners = L <= 1024 ? 8 : 4;
    return Np <= std::min<int64_t>(np_max, ffsk::kKmcMaxNp) && 64 * Np <= 3 * L && L <= kMaxLTileGram && N <= 1024 &&
           owners * ffsk::kmargc_owner_smem((int)L, (int)Np) + ffsk::align16((size_t)Np * (Np + 1)) <= kMaxSmem;
  }
  // real: any L up to 2^18 (beyond 16384 the rows of a tile are scanned in chunks of 16 per lane)
  return dtype == FFS_F64 && Np <= np_max && 64 * Np <= 3 * L && L <= kMaxLTileGram && N <= 2048 &&
         4 * ffsk::kmarg_warp_smem((int)L, (int)Np, Np <= 32, Np > 32, 32) + ffsk::align16((size_t)Np * (Np + 1)) <= kMaxSmem;
}

const void* kmc_fn(int Rl, int G) {
  if (G == 16)
    return Rl <= 1 ? reinterpret_cast<const void*>(&ffsk::ffs_kmargc_kernel<1, 4, 16>)
                   : reinterpret_cast<const void*>(&ffsk::ffs_kmargc_kernel<4, 4, 16>);
  return Rl <= 1 ? reinterpret_cast<const void*>(&ffsk::ffs_kmargc_kernel<1, 4, 32>)
       : Rl <= 4 ? reinterpret_cast<const void*>(&ffsk::ffs_kmargc_kernel<4, 4, 32>)
                 : reinterpret_cast<const void*>(&ffsk::ffs_kmargc_kernel<16, 4, 32>);
}

template <bool BLK>
const void* km_fn(int Rl, int G) {
  if (G == 16)
    return Rl <= 1 ? reinterpret_cast<const void*>(&ffsk::ffs_kmarg_kernel<1, 4, BLK, 16>)
                   : reinterpret_cast<const void*>(&ffsk::ffs_kmarg_kernel<4, 4, BLK, 16>);
  return Rl <= 1 ? reinterpret_cast<const void*>(&ffsk::ffs_kmarg_kernel<1, 4, BLK, 32>)
       : Rl <= 4 ? reinterpret_cast<const void*>(&ffsk::ffs_kmarg_kernel<4, 4, BLK, 32>)
                 : reinterpret_cast<const void*>(&ffsk::ffs_kmarg_kernel<16, 4, BLK, 32>);
}

int make_km_plan_uncached(int64_t L, int64_t N, int64_t Np, int dtype, int64_t M, KmPlan& k) {
  const bool cx = dtype == FFS_C128;
  // sample owner: a warp (32 tiles), or a half warp (16 tiles, two samples per warp) for L <= 1024,
  // where most of a draw keeps at most 16 lanes busy (C3 marginal: 0.58 -> ? ms)
  k.G = (L <= 1024 && ffsh::option(FFS_OPT_TILE_GRAM) != 4.0) ? 16 : 32;
  k.Rl = (int)((L + k.G * k.G - 1) / (k.G * k.G));
  k.Lpt = k.G * k.G * k.Rl;
  k.c_smem = Np <= 32 || cx;  // C [N'][N'] in shared memory (8 KB per warp at most), else a workspace slot per warp
  k.warps = 4;
  // N' > 32: blocked evaluation of the forms (K entries read once per block of 8 draws instead of
  // once per draw: C5 marginal 3.3 instead of 11.7 MB of K rows per sample); option value 2 / 3
  // forces flat / blocked
  const double ot = ffsh::option(FFS_OPT_TILE_GRAM);
  k.blocked = !cx && (ot == 3.0 || (ot != 2.0 && Np > 32));  // N' = 32: flat 1.91 vs blocked 2.25 ms; 48: 13.3 vs 6.9
  k.fn = cx ? kmc_fn(k.Rl, k.G) : k.blocked ? km_fn<true>(k.Rl, k.G) : km_fn<false>(k.Rl, k.G);
  k.warp_smem = cx ? ffsk::kmargc_owner_smem((int)L, (int)Np) : ffsk::kmarg_warp_smem((int)L, (int)Np, k.c_smem, k.blocked, k.G);
  const int owners = k.warps * (32 / k.G);  // per CTA
  k.smem = owners * k.warp_smem + ffsk::align16((size_t)Np * (Np + 1));  // + the entry/pair table
  if (k.smem > kMaxSmem) return fail(FFS_EINVAL, "tile-Gram path: shared memory %zu too large", k.smem);
  if (int rc = ffsh::ensure_max_smem(k.fn)) return rc;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k.fn, 32 * k.warps, k.smem) != cudaSuccess || per_sm < 1)
    return fail(FFS_EINVAL, "tile-Gram kernel does not fit on an SM (smem=%zu)", k.smem);
  const int sms = ffsh::sm_count(ffsh::device());
  int64_t ctas = (int64_t)std::min(per_sm, 8) * sms;
  ctas = std::min<int64_t>(ctas, (M + owners - 1) / owners);
  k.grid = (int)std::max<int64_t>(1, ctas);
  const size_t slots = (size_t)k.grid * owners;
  k.ws_perm = align_up((size_t)std::max<int64_t>(M, 1) * Np * 4);
  k.ws_ut = align_up((size_t)N * k.Lpt * (cx ? 16 : 8));
  k.ws_k = align_up((size_t)k.G * N * N * (cx ? 16 : 8));
  k.ws_c = k.c_smem ? 0 : align_up(slots * (size_t)Np * Np * 8);
  k.total = k.ws_perm + k.ws_ut + k.ws_k + k.ws_c;
  return FFS_OK;
}

PlanCache<KmPlan> g_km_plans;
int make_km_plan(int64_t L, int64_t N, int64_t Np, int dtype, int64_t M, KmPlan& k) {
  return g_km_plans.get(plan_key(4, L, N, Np, M, dtype), k,
                        [&](KmPlan& p) { return make_km_plan_uncached(L, N, Np, dtype, M, p); });
}

void launch_transpose(const void* U, double* Ut, int64_t L, int64_t N, int Lpt, int dtype, cudaStream_t s);

int launch_kmarg(const void* U, int64_t L, int64_t N, int dtype, int64_t M, int64_t Np, const double* uniforms,
                 int32_t* positions, int32_t* flags, void* ws, size_t ws_bytes, cudaStream_t stream, int64_t S0, int64_t S,
                 double* trace) {
  const bool cx = dtype == FFS_C128;
  KmPlan k;
  int rc = make_km_plan(L, N, Np, dtype, M, k);
  if (rc != FFS_OK) return rc;
  if (!ws || ws_bytes < k.total) return fail(FFS_ENOWS, "workspace %zu bytes < required %zu", ws_bytes, k.total);
  if (((uintptr_t)ws & (kAlign - 1)) != 0) return fail(FFS_EINVAL, "workspace not 256-byte aligned");
  char* w = static_cast<char*>(ws);
  int32_t* perm = reinterpret_cast<int32_t*>(w);
  double* Ut = reinterpret_cast<double*>(w + k.ws_perm);
  double* K = reinterpret_cast<double*>(w + k.ws_perm + k.ws_ut);
  ffsh::prof_begin(stream);
  launch_transpose(U, Ut, L, N, k.Lpt, dtype, stream);
  if (cx) {
    const dim3 kg((unsigned)((N + 31) / 32), (unsigned)((N + 31) / 32), (unsigned)k.G);
    ffsk::ffs_tile_gram_uc_kernel<<<kg, 256, 0, stream>>>(static_cast<const double*>(U), K, (int)L, (int)N, k.G * k.Rl, k.G);
  } else {
    const dim3 kg((unsigned)((N + 63) / 64), (unsigned)((N + 63) / 64), (unsigned)k.G);
    ffsk::ffs_tile_gram_u_kernel<<<kg, 256, 0, stream>>>(static_cast<const double*>(U), K, (int)L, (int)N, k.G * k.Rl, k.G);
  }
  ++ffsh::launches();
  if (int rc2 = launch_permute(uniforms, 2 * Np, perm, M, N, Np, stream)) return rc2;
  ffsk::KMargParams p{};
  p.U = static_cast<const double*>(U);
  p.Ut = Ut;
  p.K = K;
  p.permg = perm;
  p.uniforms = uniforms;
  p.positions = positions;
  p.flags = flags;
  p.Cw = k.c_smem ? nullptr : reinterpret_cast<double*>(w + k.ws_perm + k.ws_ut + k.ws_k);
  p.L = (int)L;
  p.N = (int)N;
  p.Np = (int)Np;
  p.Lpt = k.Lpt;
  p.Rl = k.Rl;
  p.M = M;
  p.S0 = S0;
  p.S = S > 0 ? S : 0;
  p.trace = S > 0 ? trace : nullptr;
  p.warp_smem = k.warp_smem;
  p.kappa_max = ffsh::option(FFS_OPT_GRAM_KAPPA);
  void* args[] = {&p};
  cudaError_t e = cudaLaunchKernel(k.fn, dim3(k.grid), dim3(32 * k.warps), args, k.smem, stream);
  if (e != cudaSuccess) return fail(FFS_ECUDA, "launch failed: %s", cudaGetErrorString(e));
  ffsh::prof_end(stream);
  ++ffsh::launches();
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

constexpr int64_t kMaxLClusterReal = 16 * 512 * 4, kMaxLClusterComplex = 16 * 512 * 2;

bool cluster_eligible(int64_t L, int dtype) {
  if (ffsh::option(FFS_OPT_FORCE_GENERIC) != 0.0 || ffsh::option(FFS_OPT_CLUSTER) == 0.0) return false;
  return L >= 2048 && L <= (dtype == FFS_C128 ? kMaxLClusterComplex : kMaxLClusterReal);
}

// cluster of CS CTAs of `threads` x R rows (CS = 2..8, or 16 with the non-portable size)
int cluster_dims(int64_t L, int rows_per_cta, int& CS) {
  CS = (int)((L + rows_per_cta - 1) / rows_per_cta);
  if (CS < 2) CS = 2;
  if (CS > 8) CS = 16;
  return CS * rows_per_cta >= L ? FFS_OK : fail(FFS_EINVAL, "L=%lld exceeds a 16-CTA cluster", (long long)L);
}

int cluster_occupancy(const void* fn, int CS, int threads, size_t smem, int& maxcl) {
  if (int rc = ffsh::ensure_max_smem(fn)) return rc;
  if (CS > 8 && cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
    return fail(FFS_ECUDA, "non-portable cluster size not allowed");
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(threads);
  cfg.gridDim = dim3(CS);
  cfg.dynamicSmemBytes = smem;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  maxcl = 0;
  if (cudaOccupancyMaxActiveClusters(&maxcl, fn, &cfg) != cudaSuccess || maxcl < 1)
    return fail(FFS_EINVAL, "cluster of %d CTAs does not fit", CS);
  return FFS_OK;
}

cudaError_t launch_cluster_kernel(const void* fn, int CS, int grid, int threads, size_t smem, cudaStream_t s,
                                  void** args) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(threads);
  cfg.gridDim = dim3(grid);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, fn, args);
}

int make_cluster_plan_uncached(int64_t L, int64_t N, int64_t Np, int dtype, int64_t M, ClusterPlan& c) {
  const bool cx = dtype == FFS_C128;
  if (cx) {
    c.fn = ffsk::cluster_kernel_ptr<cplx, 2, 8, 512>();
    c.R = 2;
  } else {
    c.fn = ffsk::cluster_kernel_ptr<double, 4, 8, 512>();
    c.R = 4;
  }
  c.B = 8;
  c.threads = 512;
  c.es = cx ? 16 : 8;
  c.Lc = c.threads * c.R;
  if (int rc = cluster_dims(L, c.Lc, c.CS)) return rc;
  c.Lpt = c.CS * c.Lc;
  c.smem = cx ? ffsk::ClusterLayout<cplx, 8>((int)N, (int)Np).total : ffsk::ClusterLayout<double, 8>((int)N, (int)Np).total;
  if (c.smem > kMaxSmem) return fail(FFS_EINVAL, "cluster path smem %zu > %zu (N'=%lld)", c.smem, kMaxSmem, (long long)Np);
  int maxcl = 0;
  if (int rc = cluster_occupancy(c.fn, c.CS, c.threads, c.smem, maxcl)) return rc;
  const int64_t ncl = std::max<int64_t>(1, std::min<int64_t>(M, maxcl));
  c.grid = (int)(ncl * c.CS);
  c.ws_ut = align_up((size_t)N * c.Lpt * c.es);
  c.ws_w = align_up((size_t)ncl * Np * Np * c.es);
  return FFS_OK;
}

PlanCache<ClusterPlan> g_cluster_plans;
int make_cluster_plan(int64_t L, int64_t N, int64_t Np, int dtype, int64_t M, ClusterPlan& c) {
  return g_cluster_plans.get(plan_key(2, L, N, Np, M, dtype), c,
                             [&](ClusterPlan& p) { return make_cluster_plan_uncached(L, N, Np, dtype, M, p); });
}

void launch_transpose(const void* U, double* Ut, int64_t L, int64_t N, int Lpt, int dtype, cudaStream_t s) {
  dim3 tb(32, 8), tg((unsigned)((Lpt + 31) / 32), (unsigned)((N + 31) / 32));
  if (dtype == FFS_C128)
    ffsk::transpose_pad_kernel<cplx><<<tg, tb, 0, s>>>(static_cast<const double*>(U), Ut, (int)L, (int)N, Lpt);
  else
    ffsk::transpose_pad_kernel<double><<<tg, tb, 0, s>>>(static_cast<const double*>(U), Ut, (int)L, (int)N, Lpt);
  ++ffsh::launches();
}

int launch_cluster(const void* U, int64_t L, int64_t N, int dtype, int64_t M, int64_t Np, const double* uniforms,
                   int32_t* positions, int32_t* flags, void* ws, size_t ws_bytes, cudaStream_t stream, int64_t S0, int64_t S,
                   double* trace) {
  ClusterPlan c;
  int rc = make_cluster_plan(L, N, Np, dtype, M, c);
  if (rc != FFS_OK) return rc;
  if (!ws || ws_bytes < c.ws_ut + c.ws_w)
    return fail(FFS_ENOWS, "workspace %zu bytes < required %zu", ws_bytes, c.ws_ut + c.ws_w);
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
  p.S0 = S0;
  p.S = S > 0 ? S : 0;
  p.trace = S > 0 ? trace : nullptr;
  launch_transpose(U, const_cast<double*>(p.Ut), L, N, c.Lpt, dtype, stream);
  void* args[] = {&p};
  ffsh::prof_begin(stream);
  cudaError_t e = launch_cluster_kernel(c.fn, c.CS, c.grid, c.threads, c.smem, stream, args);
  if (e != cudaSuccess) return fail(FFS_ECUDA, "cluster launch failed: %s", cudaGetErrorString(e));
  ffsh::prof_end(stream);
  ++ffsh::launches();
  return FFS_OK;
}

// ------------------------------------------------------------------ block-step paths
// Large L, N >= 256: per block step of B = 8 draws, one launch of the step kernel (cluster per
// sample) for a batch of S samples, then one batched Gauss-Jordan launch. Full sampling
// contracts blocks with k0 >= theta N' as ONE dense GEMM P = U Y over the batch (Ozaki-emulated
// FP64 on the INT8 tensor cores, or DMMA); marginals contract every block gathered
// (DESIGN.md §3). The ~4 launches per block are replayed as one CUDA graph.
bool dense_eligible(int64_t L, int64_t N, int64_t Np, int dtype) {
  if (ffsh::option(FFS_OPT_BLOCK_STEP) == 0.0) return false;
  // marginals (N' < N) take the same step + batched-GJ kernels with every block contracted gathered
  // (no GEMM): C5 marginal 201 -> 180 ms against the per-sample cluster kernel
  const bool marg = ffsh::option(FFS_OPT_LARGE_L_MARGINAL) != 0.0 && Np < N;
  if (ffsh::option(FFS_OPT_FORCE_GENERIC) != 0.0 || ffsh::option(FFS_OPT_CLUSTER) == 0.0) return false;
  const int64_t maxL = dtype == FFS_C128 ? kMaxLClusterComplex : kMaxLClusterReal;
  // below L = 2048 (no cluster kernel): full sampling only, every block by GEMM + Gram draws
  const int64_t minL = Np == N && ffsh::option(FFS_OPT_GRAM_DRAW) != 0.0
                           ? std::min<int64_t>(2048, (int64_t)ffsh::option(FFS_OPT_DENSE_MIN_L)) : 2048;
  return (Np == N || marg) && N >= (int64_t)ffsh::option(FFS_OPT_DENSE_MIN_N) && N % 2 == 0 && L >= minL && L <= maxL;
}

struct DensePlan {
  ClusterPlan c;
  int64_t S, ldY;      // batch, Y row stride in scalars of T
  int gemm;            // 8 / 7: Ozaki-emulated GEMM with that many slices; 0: DMMA GEMM; -1: no GEMM
  int Kp;              // GEMM K (f N) padded to the Ozaki K chunk
  size_t ws_oza, ws_ea, ws_ozb, ws_eb;
  size_t ws_perm, ws_y, ws_p, ws_w, ws_ch, ws_row, ws_ut, ws_g, total;
  int k_gather;        // blocks with k0 < k_gather contract the gathered columns in the step kernel
  int gj_pair;         // 1: the trailing Gauss-Jordan updates of two consecutive blocks in one pass
  int gram;            // 1: GEMM blocks draw on the tile Gram matrices (ffs_gram.cuh)
  int Rt;              // rows per Gram tile (32 tiles cover L)
};

template <typename T>
const void* gram_fn() { return reinterpret_cast<const void*>(&ffsk::ffs_gram_kernel<T, 8>); }
template <typename T>
const void* gram_draw_fn() { return reinterpret_cast<const void*>(&ffsk::ffs_gram_draw_kernel<T, 8>); }
template <typename T>
constexpr size_t gram_draw_smem() { return ffsk::kGramWarps * sizeof(ffsk::GramWarpSmem<T, 8>); }

// GJ tile: real 128 columns (two per thread, 16-byte W accesses), complex 64
template <typename T> constexpr int gj_tj() { return sizeof(T) == 8 ? 128 : 64; }
template <typename T>
const void* dense_gj_fn() { return reinterpret_cast<const void*>(&ffsk::ffs_dense_gj_kernel<T, 8, gj_tj<T>()>); }
template <typename T>
size_t dense_gj_bytes(int k0) { return ffsk::dense_gj_smem<T, 8, gj_tj<T>()>(k0); }
// 8-column updates (the paired schedule's eager step, the last blocks): 64 slices of i x 4 column threads
const void* dense_gj_narrow_fn() { return reinterpret_cast<const void*>(&ffsk::ffs_dense_gj_kernel<double, 8, 8, 64>); }
size_t dense_gj_narrow_bytes(int k0) { return ffsk::dense_gj_smem<double, 8, 8, 64>(k0); }
template <typename T>
const void* dense_gj2_fn() { return reinterpret_cast<const void*>(&ffsk::ffs_dense_gj2_kernel<T, 8, gj_tj<T>()>); }
template <typename T>
size_t dense_gj2_bytes(int k0) { return ffsk::dense_gj2_smem<T, 8, gj_tj<T>()>(k0); }
template <int NS>
const void* ozaki_fn() { return reinterpret_cast<const void*>(&ffsk::ffs_ozaki_gemm_kernel<NS>); }
const void* ozaki2_fn() { return reinterpret_cast<const void*>(&ffsk::ffs_ozaki_gemm2_kernel<8>); }
const void* ozaki2w_fn() { return reinterpret_cast<const void*>(&ffsk::ffs_ozaki_gemm2w_kernel); }

// 3-D tensor map [NS][rows][Kp] of int8 slices, box {kOzBK, box_rows, 1}, 64-byte swizzle
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn tensor_map_encoder() {
  // resolved once (thread-safe function-local static); first called when a plan is made, outside
  // any stream capture
  static const EncodeTiledFn enc = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess) fn = nullptr;
    return reinterpret_cast<EncodeTiledFn>(fn);
  }();
  return enc;
}

int make_dense_plan_uncached(int64_t L, int64_t N, int64_t Np, int dtype, int64_t M, DensePlan& d) {
  const bool cx = dtype == FFS_C128;
  d.c.fn = cx ? ffsk::cluster_step_kernel_ptr<cplx, 2, 8, 512>() : ffsk::cluster_step_kernel_ptr<double, 4, 8, 512>();
  d.c.R = cx ? 2 : 4;
  d.c.B = 8;
  d.c.threads = 512;
  d.c.es = cx ? 16 : 8;
  d.c.Lc = 512 * d.c.R;
  if (int rc = cluster_dims(L, d.c.Lc, d.c.CS)) return rc;
  d.c.Lpt = d.c.CS * d.c.Lc;
  d.c.smem = cx ? ffsk::ClusterLayout<cplx, 8>((int)N, (int)Np).total : ffsk::ClusterLayout<double, 8>((int)N, (int)Np).total;
  int maxcl = 0;
  if (int rc = cluster_occupancy(d.c.fn, d.c.CS, d.c.threads, d.c.smem, maxcl)) return rc;
  if (int rc = ffsh::ensure_max_smem(reinterpret_cast<const void*>(&ffsk::ffs_dgemm_kernel<32, 3>))) return rc;
  // samples per lockstep batch: as many as ~24 GB of per-sample factors W allow (larger batches =
  // larger GEMMs and fewer launches: C4 1.188 s at 1024, 1.161 s at 4096), at least 1024, at most
  // 8192 (marginals have no GEMM operands)
  const double wbytes = (double)Np * (double)Np * (cx ? 16.0 : 8.0);
  int64_t cap = std::max<int64_t>(1024, std::min<int64_t>(8192, (int64_t)(24e9 / wbytes)));
  // marginals on the Gram path keep the panels P [L][8] of a batch: at most ~4 GB of them
  const bool marg_gram = Np < N && ffsh::option(FFS_OPT_GRAM_DRAW) != 0.0 && ffsh::option(FFS_OPT_GRAM_DRAW) != 3.0 &&
                         (L + 1023) / 1024 <= ffsk::kGramMaxRl;
  if (marg_gram) cap = std::max<int64_t>(256, std::min<int64_t>(cap, (int64_t)(4e9 / ((double)L * 8 * (cx ? 16.0 : 8.0)))));
  const double ob = ffsh::option(FFS_OPT_DENSE_BATCH);
  if (ob >= 1.0) cap = (int64_t)ob;
  d.S = std::max<int64_t>(1, std::min<int64_t>(M, cap));
  // ldY in scalars of T; the GEMM's N (2 ldY real columns for complex) is a multiple of 128
  const int64_t q = cx ? ffsk::kGN / 2 : ffsk::kGN;
  d.ldY = (d.S * d.c.B + q - 1) / q * q;
  const size_t es = cx ? 16 : 8;
  const bool no_gemm = Np < N;  // marginals: gathered contraction only (the GEMM would be N/N' x wasteful)
  const int gsel = (int)ffsh::option(FFS_OPT_DENSE_GEMM);
  if (gsel != 0 && gsel != 7 && gsel != 8) return fail(FFS_EINVAL, "FFS_OPT_DENSE_GEMM must be 0, 7 or 8");
  d.gemm = no_gemm ? -1 : gsel;
  const size_t y_bytes = no_gemm ? 0 : align_up((size_t)N * d.ldY * es * (cx ? 2 : 1));  // complex: 2N x 2ldY expansion
  const size_t p_bytes = (no_gemm && !marg_gram) ? 0 : align_up((size_t)L * d.ldY * es);
  d.ws_perm = align_up((size_t)std::max<int64_t>(M, 1) * Np * 4);
  d.ws_y = y_bytes;
  d.ws_p = p_bytes;
  d.ws_w = align_up((size_t)d.S * Np * Np * es);
  d.ws_ch = align_up((size_t)d.S * (d.c.Lpt / 32) * 4);
  d.ws_row = 2 * align_up((size_t)d.S * (d.c.B * d.c.B + d.c.B) * es) + align_up((size_t)d.S * d.c.B * d.c.B * es);  // 2 x rowg, T21
  // hybrid: while k0 is small the gathered contraction (L k0 B per sample, from the transposed U)
  // costs less than the GEMM's full-N one (L N B); crossover measured on C4/C5.
  // Complex contractions do 2x the flops per gathered byte, so gathering pays longer.
  double theta;
  if (d.gemm == 0) theta = cx ? 0.6 : 0.3;
  else if (d.gemm == 7) theta = cx ? 0.35 : 0.15;
  else theta = cx ? 0.3 : 0.15;  // 8 slices, 2-SM GEMM (tools/theta_scan.py: C5 0.1-0.25, C4 0.25-0.4)
  // with the Gram draws a GEMM block costs less than a cluster-step block sooner (C5 0.1: 691.9 ms,
  // 0.15: 693.5, 0: 712.9; C4 0.2: 701.5, 0.3: 702.9, 0: 753.3; with the 32-byte U^T loads of the
  // gathered blocks C4 0.2: 663.9-666.9, 0.25: 662.1, 0.3: 660.2, 0.35: 666.3)
  if (d.gemm == 8 && ffsh::option(FFS_OPT_GRAM_DRAW) != 0.0) theta = cx ? 0.25 : 0.1;
  const double ot = ffsh::option(FFS_OPT_DENSE_THETA);
  if (ot >= 0.0) theta = ot;
  if (L < 2048) theta = 0.0;
  d.k_gather = no_gemm ? (int)Np : (int)(theta * (double)Np);
  d.ws_ut = d.k_gather > 0 ? align_up((size_t)N * d.c.Lpt * es) : 0;
  const int64_t fK = (cx ? 2 : 1) * N;
  d.Kp = (int)((fK + ffsk::kOzBK - 1) / ffsk::kOzBK * ffsk::kOzBK);
  const int64_t ncolsY = (cx ? 2 : 1) * d.ldY;
  const int ns = d.gemm > 0 ? d.gemm : 0;
  d.ws_oza = ns ? align_up((size_t)ns * L * d.Kp) : 0;
  d.ws_ea = ns ? align_up((size_t)L * 4) : 0;
  d.ws_ozb = ns ? align_up((size_t)ns * ncolsY * d.Kp) : 0;
  d.ws_eb = ns ? align_up((size_t)ncolsY * 4) : 0;
  if (ns && !tensor_map_encoder()) return fail(FFS_ECUDA, "cuTensorMapEncodeTiled unavailable");
  if (ns == 8) {
    if (int rc = ffsh::ensure_max_smem(ozaki_fn<8>())) return rc;
    if (int rc = ffsh::ensure_max_smem(ozaki2_fn())) return rc;
    if (int rc = ffsh::ensure_max_smem(ozaki2w_fn())) return rc;
  } else if (ns == 7) {
    if (int rc = ffsh::ensure_max_smem(ozaki_fn<7>())) return rc;
  }
  // Gram draws for the GEMM blocks: 32 row tiles of Rt rows (a multiple of 32) per sample
  d.gram = ((!no_gemm || marg_gram) && ffsh::option(FFS_OPT_GRAM_DRAW) != 0.0) ? 1 : 0;
  d.Rt = (int)(((L + 31) / 32 + 31) / 32 * 32);
  if (d.Rt / 32 > ffsk::kGramMaxRl) d.gram = 0;
  d.ws_g = d.gram ? align_up((size_t)d.S * (cx ? ffsk::GramIdx<cplx>::NE : ffsk::GramIdx<double>::NE) * 32 * 8) : 0;
  if (d.gram)
    if (int rc = ffsh::ensure_max_smem(cx ? gram_draw_fn<cplx>() : gram_draw_fn<double>())) return rc;
  d.total = d.ws_perm + d.ws_y + d.ws_p + d.ws_w + d.ws_ch + d.ws_row + d.ws_ut + d.ws_oza + d.ws_ea + d.ws_ozb + d.ws_eb +
            d.ws_g;
  const size_t gjs = cx ? dense_gj_bytes<cplx>((int)Np) : dense_gj_bytes<double>((int)Np);
  if (gjs > kMaxSmem) return fail(FFS_EINVAL, "block-step path: N'=%lld too large for the GJ tile", (long long)Np);
  const size_t gj2s = cx ? dense_gj2_bytes<cplx>((int)Np) : dense_gj2_bytes<double>((int)Np);
  // measured: real C5 675.2 -> 659.9 ms (the pair kernel moves half the W bytes but doubles the per-CTA
  // gathers of V[X, m_i]); complex C4 701 -> 773 ms (16 complex accumulators per column spill at 128
  // registers), so complex keeps one pass per block unless the option is 2
  const double gp = ffsh::option(FFS_OPT_GJ_PAIR);
  d.gj_pair = ((gp == 2.0 || (gp != 0.0 && !cx)) && gj2s <= kMaxSmem) ? 1 : 0;
  if (d.gj_pair)
    if (int rc = ffsh::ensure_max_smem(cx ? dense_gj2_fn<cplx>() : dense_gj2_fn<double>())) return rc;
  if (int rc = ffsh::ensure_max_smem(dense_gj_narrow_fn())) return rc;
  return ffsh::ensure_max_smem(cx ? dense_gj_fn<cplx>() : dense_gj_fn<double>());
}

PlanCache<DensePlan> g_dense_plans;
int make_dense_plan(int64_t L, int64_t N, int64_t Np, int dtype, int64_t M, DensePlan& d) {
  return g_dense_plans.get(plan_key(3, L, N, Np, M, dtype), d,
                           [&](DensePlan& p) { return make_dense_plan_uncached(L, N, Np, dtype, M, p); });
}

int oz_tensor_map(CUtensorMap* m, const int8_t* base, int ns, int64_t rows, int Kp, int box_rows) {
  const EncodeTiledFn enc = tensor_map_encoder();
  if (!enc) return fail(FFS_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[3] = {(cuuint64_t)Kp, (cuuint64_t)rows, (cuuint64_t)ns};
  const cuuint64_t strides[2] = {(cuuint64_t)Kp, (cuuint64_t)Kp * (cuuint64_t)rows};
  const cuuint32_t box[3] = {(cuuint32_t)ffsk::kOzBK, (cuuint32_t)box_rows, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  if (enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return fail(FFS_ECUDA, "cuTensorMapEncodeTiled failed");
  return FFS_OK;
}

// Issues every launch of one block-step call on `stream` (directly, or into a stream capture).
int issue_dense(const DensePlan& d, const void* U, int64_t L, int64_t N, int dtype, int64_t M, int64_t Np,
                const double* uniforms, int32_t* positions, int32_t* flags, void* ws, cudaStream_t stream, int64_t S0, int64_t S,
                double* trace) {
  const bool cx = dtype == FFS_C128;
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
  double* Gg = reinterpret_cast<double*>(ozb0 + d.ws_oza + d.ws_ea + d.ws_ozb + d.ws_eb);
  unsigned long long* gstats = nullptr;
  if (d.gram && cudaGetSymbolAddress(reinterpret_cast<void**>(&gstats), ffsk::g_gram_stats) != cudaSuccess)
    return fail(FFS_ECUDA, "cudaGetSymbolAddress failed");
  const int ns = d.gemm > 0 ? d.gemm : 0;
  const int64_t f = cx ? 2 : 1;
  const int64_t oz_ncols = f * d.ldY;
  CUtensorMap oz_ta, oz_tb;
  // the 2-SM GEMM (tcgen05 cta_group::2) for 8 slices; each CTA loads half of the B tile
  const bool oz2 = ns == 8 && ffsh::option(FFS_OPT_GEMM_2SM) != 0.0;
  // 256 x 128 pair tiles in two passes of four diagonals (ffs_ozaki_gemm2w_kernel: C5 644.5 -> 633.2 ms,
  // C4 686.1 -> 681.0 ms); option value 3: the 256 x 64 single-pass pair tiles
  const bool oz2w = oz2 && ffsh::option(FFS_OPT_GEMM_2SM) != 3.0 && oz_ncols % ffsk::kOzWBN == 0;
  if (ns) {
    if (oz_tensor_map(&oz_ta, oza, ns, L, d.Kp, ffsk::kOzBM) != FFS_OK) return FFS_ECUDA;
    if (oz_tensor_map(&oz_tb, ozb, ns, oz_ncols, d.Kp, oz2w ? ffsk::kOzWBN / 2 : oz2 ? ffsk::kOzBN / 2 : ffsk::kOzBN) != FFS_OK)
      return FFS_ECUDA;
    // A = U (real L x 2N view for complex): split once per call
    const int64_t fK = f * N;
    const unsigned g = (unsigned)((L + 7) / 8);
    if (ns == 8)
      ffsk::ffs_ozaki_split_rows_kernel<8><<<g, 256, 0, stream>>>(static_cast<const double*>(U), (int)L, (int)fK, fK, oza, d.Kp, oz_ea);
    else
      ffsk::ffs_ozaki_split_rows_kernel<7><<<g, 256, 0, stream>>>(static_cast<const double*>(U), (int)L, (int)fK, fK, oza, d.Kp, oz_ea);
    ++ffsh::launches();
  }
  if (d.k_gather > 0) launch_transpose(U, Ut, L, N, d.c.Lpt, dtype, stream);
  if (int rc = launch_permute(uniforms, 2 * Np, perm, M, N, Np, stream)) return rc;
  const void* gjf = cx ? dense_gj_fn<cplx>() : dense_gj_fn<double>();
  const int gjt = cx ? gj_tj<cplx>() : gj_tj<double>();
  double* Y = d.ws_y ? reinterpret_cast<double*>(Yb) : nullptr;
  double* Pd = reinterpret_cast<double*>(Pb);
  double* Wd = reinterpret_cast<double*>(Wb);
  const size_t rowg_bytes = align_up((size_t)d.S * (d.c.B * d.c.B + d.c.B) * es);
  double* rowg2[2] = {reinterpret_cast<double*>(rowb), reinterpret_cast<double*>(rowb + rowg_bytes)};
  double* t21 = reinterpret_cast<double*>(rowb + 2 * rowg_bytes);
  const void* gj2f = cx ? dense_gj2_fn<cplx>() : dense_gj2_fn<double>();
  for (int64_t base = 0; base < M; base += d.S) {
    const int64_t nh = std::min<int64_t>(d.S, M - base);
    if (Y && cudaMemsetAsync(Y, 0, d.ws_y, stream) != cudaSuccess) return fail(FFS_ECUDA, "memset failed");
    if (cudaMemsetAsync(ch, 0, (size_t)nh * (d.c.Lpt / 32) * 4, stream) != cudaSuccess) return fail(FFS_ECUDA, "memset failed");
    if (flags && cudaMemsetAsync(flags + base, 0, (size_t)nh * 4, stream) != cudaSuccess)
      return fail(FFS_ECUDA, "memset failed");
    if (Y) {
      const unsigned yg = (unsigned)((nh * B + 255) / 256);
      if (cx) ffsk::ffs_dense_y0_kernel<cplx, 8><<<yg, 256, 0, stream>>>(perm, Y, d.ldY, base, (int)nh, (int)Np);
      else ffsk::ffs_dense_y0_kernel<double, 8><<<yg, 256, 0, stream>>>(perm, Y, d.ldY, base, (int)nh, (int)Np);
      ++ffsh::launches();
    }
    ffsk::ClusterParams c{};
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
    c.S0 = S0;
    c.S = S > 0 ? S : 0;
    c.trace = S > 0 ? trace : nullptr;
    c.Pd = Pd;
    c.ldY = d.ldY;
    c.rowg = rowg2[0];
    c.permg = perm;
    c.chosen_g = ch;
    c.base = base;
    c.Sb = (int)nh;
    // complex: the real GEMM of U viewed as L x 2N with the real 2N x 2ldY expansion of Y
    ffsk::DgemmParams gp{};
    gp.A = static_cast<const double*>(U);
    gp.B = Y;
    gp.C = Pd;
    gp.lda = f * N;
    gp.ldb = f * d.ldY;
    gp.ldc = f * d.ldY;
    gp.M = (int)L;
    gp.N = (int)(f * d.ldY);
    gp.K = (int)(f * N);
    gp.panel = (int)(f * B);  // P in per-sample [L][B] panels (contiguous reads in the step kernel)
    ffsk::DenseGjParams q{};
    q.U = static_cast<const double*>(U);
    q.perm = perm;
    q.positions = positions;
    q.rowg = rowg2[0];
    q.W = Wd;
    q.Y = Y;
    q.ldY = d.ldY;
    q.N = (int)N;
    q.Np = (int)Np;
    q.base = base;
    const dim3 ggrid((unsigned)(f * d.ldY / ffsk::kGN), (unsigned)((L + ffsk::kGM - 1) / ffsk::kGM));
    for (int k0 = 0; k0 < Np; k0 += B) {
      // this block's pivot rows go to rowg[(k0 / B) & 1]: the paired GJ update needs two blocks' factors
      double* rowg = rowg2[(k0 / B) & 1];
      c.rowg = rowg;
      q.rowg = rowg;
      c.gather = k0 < d.k_gather ? 1 : 0;
      if (!c.gather) {
        if (ns) {
          const unsigned sg = (unsigned)(oz_ncols / 32);
          if (ns == 8)
            ffsk::ffs_ozaki_split_cols_kernel<8><<<sg, 256, 0, stream>>>(gp.B, (int)gp.K, (int)oz_ncols, gp.ldb, ozb, d.Kp, oz_eb);
          else
            ffsk::ffs_ozaki_split_cols_kernel<7><<<sg, 256, 0, stream>>>(gp.B, (int)gp.K, (int)oz_ncols, gp.ldb, ozb, d.Kp, oz_eb);
          ffsk::OzakiParams op{};
          op.ea = oz_ea;
          op.eb = oz_eb;
          op.C = gp.C;
          op.M = (int)L;
          op.N = (int)oz_ncols;
          op.K = d.Kp;
          op.panel = gp.panel;
          // stream the smaller slice set (keeps the other operand L2-resident)
          op.m_fast = (int64_t)L * d.Kp < oz_ncols * d.Kp ? 1 : 0;
          const int64_t ntiles = ((L + ffsk::kOzBM - 1) / ffsk::kOzBM) * (oz_ncols / ffsk::kOzBN);
          const dim3 og((unsigned)std::min<int64_t>(ntiles, ffsh::sm_count(ffsh::device())));  // persistent
          if (oz2w) {
            const int64_t np2 = ((L + 2 * ffsk::kOzBM - 1) / (2 * ffsk::kOzBM)) * (oz_ncols / ffsk::kOzWBN);
            const int g2 = (int)std::min<int64_t>(np2, ffsh::sm_count(ffsh::device()) / 2) * 2;  // whole pairs
            void* oargs[] = {&oz_ta, &oz_tb, &op};
            cudaError_t oe = launch_cluster_kernel(ozaki2w_fn(), 2, g2, ffsk::kOzThreads, ffsk::oz2w_smem(), stream, oargs);
            if (oe != cudaSuccess) return fail(FFS_ECUDA, "gemm launch failed: %s", cudaGetErrorString(oe));
          } else if (oz2) {
            const int64_t np2 = ((L + 2 * ffsk::kOzBM - 1) / (2 * ffsk::kOzBM)) * (oz_ncols / ffsk::kOzBN);
            const int g2 = (int)std::min<int64_t>(np2, ffsh::sm_count(ffsh::device()) / 2) * 2;  // whole pairs
            void* oargs[] = {&oz_ta, &oz_tb, &op};
            cudaError_t oe = launch_cluster_kernel(ozaki2_fn(), 2, g2, ffsk::kOzThreads, ffsk::oz2_smem<8>(), stream, oargs);
            if (oe != cudaSuccess) return fail(FFS_ECUDA, "gemm launch failed: %s", cudaGetErrorString(oe));
          } else if (ns == 8)
            ffsk::ffs_ozaki_gemm_kernel<8><<<og, ffsk::kOzThreads, ffsk::oz_smem<8>(), stream>>>(oz_ta, oz_tb, op);
          else
            ffsk::ffs_ozaki_gemm_kernel<7><<<og, ffsk::kOzThreads, ffsk::oz_smem<7>(), stream>>>(oz_ta, oz_tb, op);
          ffsh::launches() += 2;
        } else {
          ffsk::ffs_dgemm_kernel<32, 3><<<ggrid, ffsk::kGThreads, ffsk::gemm_smem<32, 3>(), stream>>>(gp);
          ++ffsh::launches();
        }
      }
      c.k0 = k0;
      cudaError_t e;
      // gathered blocks of a full-sampling call with the Gram draws: the cluster kernel only contracts
      // the panel (into the GEMM's output buffer), the draws run on the Gram path like a GEMM block
      const bool panel_only = c.gather && d.gram && d.ws_p > 0 && ffsh::option(FFS_OPT_GRAM_DRAW) != 3.0;
      c.panel_out = panel_only ? 1 : 0;
      if (panel_only) {
        void* args[] = {&c};
        e = launch_cluster_kernel(d.c.fn, d.c.CS, (int)(nh * d.c.CS), d.c.threads, d.c.smem, stream, args);
        if (e != cudaSuccess) return fail(FFS_ECUDA, "panel launch failed: %s", cudaGetErrorString(e));
        ++ffsh::launches();
      }
      if ((!c.gather || panel_only) && d.gram) {
        // draws on the tile Gram matrices of the GEMM panel: one pass over P, then a warp per sample
        ffsk::GramParams g{};
        g.Pd = Pd;
        g.G = Gg;
        g.chosen_g = ch;
        g.uniforms = uniforms;
        g.positions = positions;
        g.flags = flags;
        g.rowg = rowg;
        g.L = (int)L;
        g.Lpt = d.c.Lpt;
        g.Np = (int)Np;
        g.Sb = (int)nh;
        g.Rt = d.Rt;
        g.k0 = k0;
        g.base = base;
        g.S0 = S0;
        g.S = S > 0 ? S : 0;
        g.trace = S > 0 ? trace : nullptr;
        g.stats = gstats;
        g.kappa_max = ffsh::option(FFS_OPT_GRAM_KAPPA);
        void* gargs[] = {&g};
        e = cudaLaunchKernel(cx ? gram_fn<cplx>() : gram_fn<double>(), dim3((unsigned)((nh * 32 + 7) / 8)), dim3(256), gargs, 0,
                             stream);
        if (e != cudaSuccess) return fail(FFS_ECUDA, "gram launch failed: %s", cudaGetErrorString(e));
        e = cudaLaunchKernel(cx ? gram_draw_fn<cplx>() : gram_draw_fn<double>(),
                             dim3((unsigned)((nh + ffsk::kGramWarps - 1) / ffsk::kGramWarps)), dim3(32 * ffsk::kGramWarps), gargs,
                             cx ? gram_draw_smem<cplx>() : gram_draw_smem<double>(), stream);
        if (e != cudaSuccess) return fail(FFS_ECUDA, "gram draw launch failed: %s", cudaGetErrorString(e));
        ffsh::launches() += 2;
      } else {
        void* args[] = {&c};
        e = launch_cluster_kernel(d.c.fn, d.c.CS, (int)(nh * d.c.CS), d.c.threads, d.c.smem, stream, args);
        if (e != cudaSuccess) return fail(FFS_ECUDA, "step launch failed: %s", cudaGetErrorString(e));
        ++ffsh::launches();
      }
      // Gauss-Jordan update. Paired mode: an even block e (k0 = 2 B p) with later columns beyond the
      // next block only updates that next block's B columns; after the odd block both blocks'
      // trailing updates run in one pass over W (ffs_dense_gj2_kernel)
      const bool even = ((k0 / B) & 1) == 0;
      const bool pair_first = d.gj_pair && even && k0 + 2 * B < Np;
      const bool pair_second = d.gj_pair && !even && k0 + B < Np;
      if (pair_second) {
        const int ke = k0 - B;  // the pair starts at the even block
        if (cx)
          ffsk::ffs_dense_t21_kernel<cplx, 8><<<(unsigned)nh, 256, 0, stream>>>(static_cast<const double*>(U), perm, positions, Wd,
                                                                               t21, base, (int)N, (int)Np, ke);
        else
          ffsk::ffs_dense_t21_kernel<double, 8><<<(unsigned)nh, 256, 0, stream>>>(static_cast<const double*>(U), perm, positions,
                                                                                 Wd, t21, base, (int)N, (int)Np, ke);
        ffsk::DenseGj2Params q2{};
        q2.U = static_cast<const double*>(U);
        q2.perm = perm;
        q2.positions = positions;
        q2.rowg1 = rowg2[(ke / B) & 1];
        q2.rowg2 = rowg;
        q2.t21 = t21;
        q2.W = Wd;
        q2.Y = Y;
        q2.ldY = d.ldY;
        q2.base = base;
        q2.N = (int)N;
        q2.Np = (int)Np;
        q2.k0 = ke;
        const int nc = (int)Np - ke - 2 * B;
        const dim3 jg((unsigned)((nc + gjt - 1) / gjt), (unsigned)nh);
        const size_t gsm = cx ? dense_gj2_bytes<cplx>(ke) : dense_gj2_bytes<double>(ke);
        void* qargs[] = {&q2};
        e = cudaLaunchKernel(gj2f, jg, dim3(256), qargs, gsm, stream);
        if (e != cudaSuccess) return fail(FFS_ECUDA, "gj2 launch failed: %s", cudaGetErrorString(e));
        ffsh::launches() += 2;
      } else if (k0 + B < Np) {
        q.k0 = k0;
        q.jend = pair_first ? k0 + 2 * B : (int)Np;
        const int nc = q.jend - k0 - B;
        const bool narrow = !cx && nc <= 8 && dense_gj_narrow_bytes(k0) <= kMaxSmem;
        const dim3 jg(narrow ? 1u : (unsigned)((nc + gjt - 1) / gjt), (unsigned)nh);
        const size_t gsm = narrow ? dense_gj_narrow_bytes(k0) : cx ? dense_gj_bytes<cplx>(k0) : dense_gj_bytes<double>(k0);
        void* qargs[] = {&q};
        e = cudaLaunchKernel(narrow ? dense_gj_narrow_fn() : gjf, jg, dim3(256), qargs, gsm, stream);
        if (e != cudaSuccess) return fail(FFS_ECUDA, "gj launch failed: %s", cudaGetErrorString(e));
        ++ffsh::launches();
      }
    }
  }
  return FFS_OK;
}

// CUDA-graph driver (north_star (d)): a multi-launch schedule is captured once per (arguments,
// options) and replayed with one cudaGraphLaunch; a change of pointers or sizes re-captures and
// updates the executable graph in place. Per host thread, the last few argument sets are kept.
// Capture happens on a library-owned stream (the caller's may be the legacy default stream, which
// cannot be captured); the executable is launched on the caller's stream. When the caller's stream
// is itself being captured, or the option is off, the launches are issued directly.
struct GraphEntry {
  std::vector<int64_t> key;
  cudaGraphExec_t exec = nullptr;
  int launches = 0;
};
thread_local GraphEntry g_graphs[8];
thread_local unsigned g_graph_next = 0;
thread_local cudaStream_t g_capture_stream = nullptr;

template <typename Issue>
int run_graph(const std::vector<int64_t>& key0, cudaStream_t stream, Issue&& issue) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess) return fail(FFS_ECUDA, "cudaStreamIsCapturing failed");
  if (ffsh::option(FFS_OPT_GRAPH) == 0.0 || cs != cudaStreamCaptureStatusNone) {
    ffsh::prof_begin(stream);
    const int rc = issue(stream);
    ffsh::prof_end(stream);
    return rc;
  }
  std::vector<int64_t> key = key0;
  key.push_back((int64_t)ffsh::options_version());
  key.push_back(ffsh::device());
  GraphEntry* ge = nullptr;
  for (auto& g : g_graphs)
    if (g.exec && g.key == key) ge = &g;
  if (!ge) {
    ge = &g_graphs[g_graph_next++ % 8];
    if (!g_capture_stream && cudaStreamCreateWithFlags(&g_capture_stream, cudaStreamNonBlocking) != cudaSuccess)
      return fail(FFS_ECUDA, "capture stream creation failed");
    cudaGraph_t graph_def = nullptr;
    if (cudaStreamBeginCapture(g_capture_stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
      return fail(FFS_ECUDA, "cudaStreamBeginCapture failed");
    const int l0 = ffsh::launches();
    const int rc = issue(g_capture_stream);
    const cudaError_t ce = cudaStreamEndCapture(g_capture_stream, &graph_def);
    if (rc != FFS_OK) {
      if (graph_def) cudaGraphDestroy(graph_def);
      return rc;
    }
    if (ce != cudaSuccess || !graph_def) return fail(FFS_ECUDA, "stream capture failed: %s", cudaGetErrorString(ce));
    bool updated = false;
    if (ge->exec) {
      cudaGraphExecUpdateResultInfo info;
      updated = cudaGraphExecUpdate(ge->exec, graph_def, &info) == cudaSuccess;
      if (!updated) {
        cudaGetLastError();
        cudaGraphExecDestroy(ge->exec);
        ge->exec = nullptr;
      }
    }
    if (!updated && cudaGraphInstantiate(&ge->exec, graph_def, 0) != cudaSuccess) {
      cudaGraphDestroy(graph_def);
      ge->exec = nullptr;
      return fail(FFS_ECUDA, "cudaGraphInstantiate failed");
    }
    cudaGraphDestroy(graph_def);
    ge->key = key;
    ge->launches = ffsh::launches() - l0;
  } else {
    ffsh::launches() += ge->launches;
  }
  ffsh::prof_begin(stream);
  const cudaError_t e = cudaGraphLaunch(ge->exec, stream);
  if (e != cudaSuccess) return fail(FFS_ECUDA, "cudaGraphLaunch failed: %s", cudaGetErrorString(e));
  ffsh::prof_end(stream);
  return FFS_OK;
}

int launch_dense(const void* U, int64_t L, int64_t N, int dtype, int64_t M, int64_t Np, const double* uniforms,
                 int32_t* positions, int32_t* flags, void* ws, size_t ws_bytes, cudaStream_t stream, int64_t S0, int64_t S,
                 double* trace) {
  DensePlan d;
  int rc = make_dense_plan(L, N, Np, dtype, M, d);
  if (rc != FFS_OK) return rc;
  if (!ws || ws_bytes < d.total) return fail(FFS_ENOWS, "workspace %zu bytes < required %zu", ws_bytes, d.total);
  if (((uintptr_t)ws & (kAlign - 1)) != 0) return fail(FFS_EINVAL, "workspace not 256-byte aligned");
  const std::vector<int64_t> key = {1, (int64_t)(uintptr_t)U, L, N, dtype, M, Np, (int64_t)(uintptr_t)uniforms,
                                    (int64_t)(uintptr_t)positions, (int64_t)(uintptr_t)flags, (int64_t)(uintptr_t)ws,
                                    S0, S, (int64_t)(uintptr_t)trace};
  return run_graph(key, stream, [&](cudaStream_t s) {
    return issue_dense(d, U, L, N, dtype, M, Np, uniforms, positions, flags, ws, s, S0, S, trace);
  });
}

// ------------------------------------------------------------------ generic CTA/warp-owner path
int launch_generic(const void* U, int64_t L, int64_t N, int dtype, int64_t M, int64_t Np, const double* uniforms,
                   int32_t* positions, int32_t* flags, void* ws, size_t ws_bytes, cudaStream_t stream, int64_t S0, int64_t S,
                   double* trace) {
  Plan pl;
  int rc = make_plan(L, N, Np, dtype, M, pl);
  if (rc != FFS_OK) return rc;
  const size_t need = pl.ws_ut + pl.ws_wfull;
  if (need > 0 && (!ws || ws_bytes < need))
    return fail(FFS_ENOWS, "workspace %zu bytes < required %zu", ws_bytes, need);
  if (((uintptr_t)ws & (kAlign - 1)) != 0) return fail(FFS_EINVAL, "workspace not 256-byte aligned");
  char* w = static_cast<char*>(ws);
  ffsk::Params p{};
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
  p.S0 = S0;
  p.S = S > 0 ? S : 0;
  p.trace = S > 0 ? trace : nullptr;
  p.owner_smem = pl.owner_smem;
  p.ushared_smem = pl.ushared_smem;
  p.ustride = (int)(2 * Np);
  p.usel = (int)Np;
  if (!pl.v.usmem) launch_transpose(U, const_cast<double*>(p.Ut), L, N, pl.Lp, dtype, stream);
  void* args[] = {&p};
  ffsh::prof_begin(stream);
  cudaError_t e = cudaLaunchKernel(pl.v.fn, dim3(pl.grid), dim3(pl.threads), args, pl.smem, stream);
  if (e != cudaSuccess) return fail(FFS_ECUDA, "launch failed: %s", cudaGetErrorString(e));
  ffsh::prof_end(stream);
  ++ffsh::launches();
  return FFS_OK;
}

int check_shape(int64_t L, int64_t N, int64_t Np, int dtype, int64_t M, bool tile_gram_ok = false) {
  if (L < 1 || N < 1 || N > L || Np < 1 || Np > N || L > INT32_MAX || M < 0)
    return fail(FFS_EINVAL, "invalid shape L=%lld N=%lld N'=%lld M=%lld", (long long)L, (long long)N, (long long)Np,
                (long long)M);
  if (dtype != FFS_F64 && dtype != FFS_C128) return fail(FFS_EINVAL, "unknown dtype %d", dtype);
  const int64_t maxL = dtype == FFS_C128 ? kMaxLComplex : kMaxLReal;
  if (L > maxL && !(tile_gram_ok && kmarg_eligible(L, N, Np, dtype)))  // (the tile-Gram path keeps no panel: small-N' calls up to L = 2^18)
    return fail(FFS_EINVAL, "unsupported L=%lld for dtype %d: the per-sample panel must fit one SM's registers "
                "(max L %lld; real U with small N' up to %lld on the tile-Gram path); see include/ffs.h", (long long)L, dtype,
                (long long)maxL, (long long)kMaxLTileGram);
  return FFS_OK;
}

int launch(const void* U, int64_t L, int64_t N, int dtype, int64_t M, int64_t Np, const double* uniforms,
           int32_t* positions, int32_t* flags, void* ws, size_t ws_bytes, cudaStream_t stream, int64_t S0, int64_t S,
           double* trace) {
  ffsh::launches() = 0;
  if (M == 0) return FFS_OK;
  if (int rc = check_shape(L, N, Np, dtype, M, true)) return rc;
  if (!U || !uniforms || !positions) return fail(FFS_EINVAL, "null U/uniforms/positions with M=%lld", (long long)M);
  if (S > 0 && !trace) return fail(FFS_EINVAL, "null trace buffer with S=%lld", (long long)S);
  int rc;
  if (warp_eligible(L, N, Np, dtype))
    rc = launch_warp(U, L, N, M, Np, uniforms, positions, flags, ws, ws_bytes, stream, S0, S, trace);
  else if (kmarg_eligible(L, N, Np, dtype))
    rc = launch_kmarg(U, L, N, dtype, M, Np, uniforms, positions, flags, ws, ws_bytes, stream, S0, S, trace);
  else if (dense_eligible(L, N, Np, dtype))
    rc = launch_dense(U, L, N, dtype, M, Np, uniforms, positions, flags, ws, ws_bytes, stream, S0, S, trace);
  else if (cluster_eligible(L, dtype))
    rc = launch_cluster(U, L, N, dtype, M, Np, uniforms, positions, flags, ws, ws_bytes, stream, S0, S, trace);
  else
    rc = launch_generic(U, L, N, dtype, M, Np, uniforms, positions, flags, ws, ws_bytes, stream, S0, S, trace);
  if (rc != FFS_OK) return rc;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(FFS_ECUDA, "CUDA error: %s", cudaGetErrorString(e));
  ffsh::clear_error();
  return FFS_OK;
}

size_t workspace_bytes(int64_t L, int64_t N, int64_t Np, int dtype, int64_t M) {
  if (check_shape(L, N, Np, dtype, std::max<int64_t>(M, 1), true) != FFS_OK) return 0;
  M = std::max<int64_t>(M, 1);
  if (warp_eligible(L, N, Np, dtype)) {
    WarpPlan w;
    return make_warp_plan(L, N, Np, M, w) == FFS_OK ? w.ws_perm : 0;
  }
  if (kmarg_eligible(L, N, Np, dtype)) {
    KmPlan k;
    return make_km_plan(L, N, Np, dtype, M, k) == FFS_OK ? k.total : 0;
  }
  if (dense_eligible(L, N, Np, dtype)) {
    DensePlan d;
    return make_dense_plan(L, N, Np, dtype, M, d) == FFS_OK ? d.total : 0;
  }
  if (cluster_eligible(L, dtype)) {
    ClusterPlan c;
    return make_cluster_plan(L, N, Np, dtype, M, c) == FFS_OK ? c.ws_ut + c.ws_w : 0;
  }
  Plan pl;
  return make_plan(L, N, Np, dtype, M, pl) == FFS_OK ? pl.ws_ut + pl.ws_wfull : 0;
}


// ------------------------------------------------------------------ L-ensemble front end
// ffs_lens_prep_kernel (keep draws + permutation of the kept columns) then ffs_sample_kernel in
// ragged mode (each sample its own N_i <= K steps). Workspace: [cols M x K | nps M | generic plan].
struct LensLayout {
  size_t cols, nps, plan, total;
  Plan pl;
  int prep_tpb;
};
int lens_layout(int64_t L, int64_t K, int dtype, int64_t M, LensLayout& y) {
  if (int rc = check_shape(L, K, K, dtype, std::max<int64_t>(M, 1))) return rc;
  if (int rc = make_plan(L, K, K, dtype, std::max<int64_t>(M, 1), y.pl)) return rc;
  y.cols = 0;
  y.nps = align_up((size_t)std::max<int64_t>(M, 1) * K * 4);
  y.plan = y.nps + align_up((size_t)std::max<int64_t>(M, 1) * 4);
  y.total = y.plan + y.pl.ws_ut + y.pl.ws_wfull;
  y.prep_tpb = (int)std::max<int64_t>(1, std::min<int64_t>(128, 40960 / (4 * K)));
  return FFS_OK;
}

int launch_lensemble(const void* V, const double* lambda, int64_t L, int64_t K, int dtype, int64_t M,
                     const double* uniforms, int32_t* positions, int32_t* counts, int32_t* flags, void* ws,
                     size_t ws_bytes, cudaStream_t stream) {
  ffsh::launches() = 0;
  if (M == 0) return FFS_OK;
  if (M < 0) return fail(FFS_EINVAL, "M=%lld < 0", (long long)M);
  if (!V || !lambda || !uniforms || !positions) return fail(FFS_EINVAL, "null V/lambda/uniforms/positions");
  LensLayout y;
  if (int rc = lens_layout(L, K, dtype, M, y)) return rc;
  if (!ws || ws_bytes < y.total) return fail(FFS_ENOWS, "workspace %zu bytes < required %zu", ws_bytes, y.total);
  if (((uintptr_t)ws & (kAlign - 1)) != 0) return fail(FFS_EINVAL, "workspace not 256-byte aligned");
  char* w = static_cast<char*>(ws);
  int32_t* cols = reinterpret_cast<int32_t*>(w + y.cols);
  int32_t* nps = reinterpret_cast<int32_t*>(w + y.nps);
  char* pw = w + y.plan;
  const Plan& pl = y.pl;
  const int64_t pgrid = (M + y.prep_tpb - 1) / y.prep_tpb;
  ffsk::ffs_lens_prep_kernel<<<(unsigned)pgrid, y.prep_tpb, (size_t)y.prep_tpb * K * 4, stream>>>(lambda, uniforms, cols,
                                                                                              nps, M, (int)K);
  ++ffsh::launches();
  ffsk::Params p{};
  p.U = static_cast<const double*>(V);
  p.Ut = pl.v.usmem ? nullptr : reinterpret_cast<const double*>(pw);
  p.L = (int)L;
  p.N = (int)K;
  p.Np = (int)K;
  p.Lp = pl.Lp;
  p.ut_stride = pl.ut_stride;
  p.M = M;
  p.uniforms = uniforms;
  p.positions = positions;
  p.flags = flags;
  p.wfull = reinterpret_cast<double*>(pw + pl.ws_ut);
  p.owner_smem = pl.owner_smem;
  p.ushared_smem = pl.ushared_smem;
  p.cols = cols;
  p.nps = nps;
  p.ustride = (int)(3 * K);
  p.usel = (int)(2 * K);
  if (!pl.v.usmem) launch_transpose(V, const_cast<double*>(p.Ut), L, K, pl.Lp, dtype, stream);
  void* args[] = {&p};
  ffsh::prof_begin(stream);
  cudaError_t e = cudaLaunchKernel(pl.v.fn, dim3(pl.grid), dim3(pl.threads), args, pl.smem, stream);
  if (e != cudaSuccess) return fail(FFS_ECUDA, "launch failed: %s", cudaGetErrorString(e));
  ffsh::prof_end(stream);
  ++ffsh::launches();
  if (counts && cudaMemcpyAsync(counts, nps, (size_t)M * 4, cudaMemcpyDeviceToDevice, stream) != cudaSuccess)
    return fail(FFS_ECUDA, "counts copy failed");
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(FFS_ECUDA, "CUDA error: %s", cudaGetErrorString(e));
  ffsh::clear_error();
  return FFS_OK;
}

// ------------------------------------------------------------------ Supp S7 Metropolis variant
// ffs_permute_kernel (a1) then ffs_metro_kernel (one warp per sample, W per warp slot).
// Workspace: [perm M x N' | W slots x N'^2].
struct MetroLayout {
  size_t perm, wbuf, total, smem;
  int grid;
};
int metro_layout(int64_t L, int64_t N, int64_t Np, int64_t Mc, int dtype, int64_t M, MetroLayout& y) {
  if (L < 1 || N < 1 || N > L || Np < 1 || Np > N || L > INT32_MAX || M < 0 || Mc < 0 || Mc > 4096)
    return fail(FFS_EINVAL, "invalid shape L=%lld N=%lld N'=%lld M_cond=%lld", (long long)L, (long long)N,
                (long long)Np, (long long)Mc);
  if (dtype != FFS_F64 && dtype != FFS_C128) return fail(FFS_EINVAL, "unknown dtype %d", dtype);
  const bool cx = dtype == FFS_C128;
  const size_t es = cx ? 16 : 8;
  y.smem = (size_t)ffsk::kMetroWarps * (cx ? ffsk::metro_warp_smem<cplx>((int)Np, (int)Mc, (int)N)
                                           : ffsk::metro_warp_smem<double>((int)Np, (int)Mc, (int)N));
  if (y.smem > kMaxSmem) return fail(FFS_EINVAL, "N'=%lld / M_cond=%lld too large for the Metropolis kernel",
                                     (long long)Np, (long long)Mc);
  const void* fn = cx ? reinterpret_cast<const void*>(&ffsk::ffs_metro_kernel<cplx>)
                      : reinterpret_cast<const void*>(&ffsk::ffs_metro_kernel<double>);
  if (int rc = ffsh::ensure_max_smem(fn)) return rc;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, ffsk::kMetroWarps * 32, y.smem) != cudaSuccess ||
      per_sm < 1)
    return fail(FFS_EINVAL, "Metropolis kernel does not fit on an SM");
  const int64_t M1 = std::max<int64_t>(M, 1);
  y.grid = (int)std::max<int64_t>(1, std::min<int64_t>((M1 + ffsk::kMetroWarps - 1) / ffsk::kMetroWarps,
                                                       (int64_t)per_sm * ffsh::sm_count(ffsh::device())));
  y.perm = 0;
  y.wbuf = align_up((size_t)M1 * Np * 4);
  y.total = y.wbuf + align_up((size_t)y.grid * ffsk::kMetroWarps * Np * Np * es);
  return FFS_OK;
}

int launch_metropolis(const void* U, int64_t L, int64_t N, int dtype, int64_t M, int64_t Np, int64_t Mc,
                      const double* uniforms, int32_t* positions, int32_t* flags, void* ws, size_t ws_bytes,
                      cudaStream_t stream) {
  ffsh::launches() = 0;
  if (M == 0) return FFS_OK;
  if (!U || !uniforms || !positions) return fail(FFS_EINVAL, "null U/uniforms/positions");
  MetroLayout y;
  if (int rc = metro_layout(L, N, Np, Mc, dtype, M, y)) return rc;
  if (!ws || ws_bytes < y.total) return fail(FFS_ENOWS, "workspace %zu bytes < required %zu", ws_bytes, y.total);
  if (((uintptr_t)ws & (kAlign - 1)) != 0) return fail(FFS_EINVAL, "workspace not 256-byte aligned");
  char* w = static_cast<char*>(ws);
  int32_t* perm = reinterpret_cast<int32_t*>(w + y.perm);
  const int64_t ustride = Np + Np * (1 + 2 * Mc);
  if (int rc = launch_permute(uniforms, ustride, perm, M, N, Np, stream)) return rc;
  ffsk::MetroParams p{};
  p.U = static_cast<const double*>(U);
  p.perm = perm;
  p.uniforms = uniforms;
  p.positions = positions;
  p.flags = flags;
  p.wbuf = reinterpret_cast<double*>(w + y.wbuf);
  p.M = M;
  p.L = (int)L;
  p.N = (int)N;
  p.Np = (int)Np;
  p.Mc = (int)Mc;
  ffsh::prof_begin(stream);
  if (dtype == FFS_C128)
    ffsk::ffs_metro_kernel<cplx><<<y.grid, ffsk::kMetroWarps * 32, y.smem, stream>>>(p);
  else
    ffsk::ffs_metro_kernel<double><<<y.grid, ffsk::kMetroWarps * 32, y.smem, stream>>>(p);
  ffsh::prof_end(stream);
  ++ffsh::launches();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(FFS_ECUDA, "CUDA error: %s", cudaGetErrorString(e));
  ffsh::clear_error();
  return FFS_OK;
}

// ------------------------------------------------------------------ modified-HKPV comparator
// Lockstep batches of S samples: per step one ffs_hkpv_step_kernel launch (CTA per sample: draw +
// Gram-Schmidt) and one DMMA GEMM with the residual-update epilogue; replayed as a CUDA graph.
// Workspace: [U padded L x ldu | r S x L | chosen | E S x N' x N | Eb].
struct HkpvPlan {
  int64_t S, ldu, ldE, fK;
  size_t u, r, ch, e, eb, total, step_smem;
};
int hkpv_plan(int64_t L, int64_t N, int64_t Np, int dtype, int64_t M, HkpvPlan& h) {
  if (int rc = check_shape(L, N, Np, dtype, std::max<int64_t>(M, 1))) return rc;
  const bool cx = dtype == FFS_C128;
  const size_t es = cx ? 16 : 8;
  const int64_t f = cx ? 2 : 1;
  h.ldu = cx ? N : ((N + 1) & ~int64_t(1));  // 16-byte aligned rows of the GEMM's A operand
  h.fK = f * h.ldu;
  // batch: residuals, e-vectors and the GEMM operand of S samples within ~16 GB
  const double per = (double)L * 8 + (double)Np * N * es + (double)f * h.fK * 8 + ((L + 31) / 32) * 4.0;
  h.S = std::max<int64_t>(1, std::min<int64_t>(std::max<int64_t>(M, 1), (int64_t)(16e9 / per)));
  const double ob = ffsh::option(FFS_OPT_DENSE_BATCH);
  if (ob >= 1.0) h.S = std::min<int64_t>(h.S, (int64_t)ob);
  const int64_t q = ffsk::kGN / f;
  h.ldE = (h.S + q - 1) / q * q;
  h.u = 0;
  h.r = align_up((size_t)L * h.ldu * es);
  h.ch = h.r + align_up((size_t)h.S * L * 8);
  h.e = h.ch + align_up((size_t)h.S * ((L + 31) / 32) * 4);
  h.eb = h.e + align_up((size_t)h.S * Np * N * es);
  h.total = h.eb + align_up((size_t)h.fK * f * h.ldE * 8);
  h.step_smem = 32 * 8 + 96 * 4 + (size_t)(N + Np) * es;
  if (h.step_smem > kMaxSmem || N > 16384) return fail(FFS_EINVAL, "N=%lld too large for the HKPV step kernel", (long long)N);
  const void* sf = cx ? reinterpret_cast<const void*>(&ffsk::ffs_hkpv_step_kernel<cplx>)
                      : reinterpret_cast<const void*>(&ffsk::ffs_hkpv_step_kernel<double>);
  if (int rc = ffsh::ensure_max_smem(sf)) return rc;
  return ffsh::ensure_max_smem(reinterpret_cast<const void*>(&ffsk::ffs_dgemm_kernel<32, 3, 1>));
}

int issue_hkpv(const HkpvPlan& h, const void* U, int64_t L, int64_t N, int dtype, int64_t M, int64_t Np,
               const double* uniforms, int32_t* positions, int32_t* flags, void* ws, cudaStream_t s) {
  const bool cx = dtype == FFS_C128;
  const size_t es = cx ? 16 : 8;
  const int64_t f = cx ? 2 : 1;
  char* w = static_cast<char*>(ws);
  double* Up = reinterpret_cast<double*>(w + h.u);
  if (cudaMemcpy2DAsync(Up, h.ldu * es, U, N * es, N * es, L, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return fail(FFS_ECUDA, "U copy failed");
  if (h.ldu > N && cudaMemset2DAsync(reinterpret_cast<char*>(Up) + N * es, h.ldu * es, 0, (h.ldu - N) * es, L, s) != cudaSuccess)
    return fail(FFS_ECUDA, "U pad failed");
  ffsk::HkpvParams p{};
  p.U = Up;
  p.ldu = h.ldu;
  p.uniforms = uniforms;
  p.positions = positions;
  p.flags = flags;
  p.r = reinterpret_cast<double*>(w + h.r);
  p.chosen = reinterpret_cast<uint32_t*>(w + h.ch);
  p.E = reinterpret_cast<double*>(w + h.e);
  p.Eb = reinterpret_cast<double*>(w + h.eb);
  p.ldE = h.ldE;
  p.L = (int)L;
  p.N = (int)N;
  p.Np = (int)Np;
  ffsk::DgemmParams gp{};
  gp.A = Up;
  gp.B = p.Eb;
  gp.C = nullptr;
  gp.lda = h.fK;
  gp.ldb = f * h.ldE;
  gp.ldc = 0;
  gp.M = (int)L;
  gp.N = (int)(f * h.ldE);
  gp.K = (int)h.fK;
  gp.panel = 0;
  gp.r = p.r;
  gp.rld = L;
  gp.cplx = cx ? 1 : 0;
  const dim3 ggrid((unsigned)(f * h.ldE / ffsk::kGN), (unsigned)((L + ffsk::kGM - 1) / ffsk::kGM));
  for (int64_t base = 0; base < M; base += h.S) {
    const int64_t Sb = std::min<int64_t>(h.S, M - base);
    p.base = base;
    p.Sb = (int)Sb;
    gp.nsamp = (int)Sb;
    if (cudaMemsetAsync(p.Eb, 0, (size_t)h.fK * f * h.ldE * 8, s) != cudaSuccess) return fail(FFS_ECUDA, "memset failed");
    const unsigned ig = (unsigned)std::min<int64_t>((Sb * L + 255) / 256, 65535);
    if (cx) ffsk::ffs_hkpv_init_kernel<cplx><<<ig, 256, 0, s>>>(p);
    else ffsk::ffs_hkpv_init_kernel<double><<<ig, 256, 0, s>>>(p);
    ++ffsh::launches();
    for (int k = 0; k < Np; ++k) {
      p.k = k;
      if (cx) ffsk::ffs_hkpv_step_kernel<cplx><<<(unsigned)Sb, ffsk::kHkpvThreads, h.step_smem, s>>>(p);
      else ffsk::ffs_hkpv_step_kernel<double><<<(unsigned)Sb, ffsk::kHkpvThreads, h.step_smem, s>>>(p);
      ++ffsh::launches();
      if (k + 1 < Np) {
        ffsk::ffs_dgemm_kernel<32, 3, 1><<<ggrid, ffsk::kGThreads, ffsk::gemm_smem<32, 3>(), s>>>(gp);
        ++ffsh::launches();
      }
    }
  }
  return FFS_OK;
}

// small real L: the fused warp-per-sample kernel (U^T and e-vectors in shared memory)
struct HkpvWarpPlan {
  const void* fn;
  int R, maxt, warps, grid, Lp, ut_stride;
  size_t ushared, owner, smem;
};
template <int R, int MAXT>
void hkpv_warp_fn(HkpvWarpPlan& w) {
  w.fn = reinterpret_cast<const void*>(&ffsk::ffs_hkpv_warp_kernel<R, MAXT>);
  w.R = R;
  w.maxt = MAXT;
}
bool hkpv_warp_plan(int64_t L, int64_t N, int64_t Np, int dtype, int64_t M, HkpvWarpPlan& w) {
  if (dtype != FFS_F64 || L > 256 || ffsh::option(FFS_OPT_FORCE_GENERIC) != 0.0) return false;
  if (L <= 32) hkpv_warp_fn<1, 512>(w);
  else if (L <= 64) hkpv_warp_fn<2, 512>(w);
  else if (L <= 128) hkpv_warp_fn<4, 512>(w);
  else hkpv_warp_fn<8, 512>(w);
  w.Lp = 32 * w.R;
  w.ut_stride = w.Lp + 2;
  w.ushared = ffsk::align16((size_t)N * w.ut_stride * 8);
  w.owner = ffsk::hkpv_warp_owner_bytes((int)N, (int)Np);
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, w.fn) != cudaSuccess) return false;
  const int by_regs = 4 * std::max(1, 16384 / (((std::max(fa.numRegs, 1) * 32 + 255) / 256) * 256));
  int warps = std::min(w.maxt / 32, by_regs);
  while (warps > 1 && w.ushared + (size_t)warps * w.owner > kMaxSmem) --warps;
  w.warps = warps;
  w.smem = w.ushared + (size_t)warps * w.owner;
  if (w.smem > kMaxSmem || ffsh::ensure_max_smem(w.fn) != FFS_OK) return false;
  const int64_t ctas = (std::max<int64_t>(M, 1) + warps - 1) / warps;
  w.grid = (int)std::max<int64_t>(1, std::min<int64_t>(ctas, ffsh::sm_count(ffsh::device())));
  return true;
}

int launch_hkpv(const void* U, int64_t L, int64_t N, int dtype, int64_t M, int64_t Np, const double* uniforms,
                int32_t* positions, int32_t* flags, void* ws, size_t ws_bytes, cudaStream_t stream) {
  ffsh::launches() = 0;
  if (M == 0) return FFS_OK;
  if (!U || !uniforms || !positions) return fail(FFS_EINVAL, "null U/uniforms/positions");
  if (int rc = check_shape(L, N, Np, dtype, M)) return rc;
  HkpvWarpPlan wp;
  if (hkpv_warp_plan(L, N, Np, dtype, M, wp)) {
    ffsk::HkpvWarpParams q{};
    q.U = static_cast<const double*>(U);
    q.uniforms = uniforms;
    q.positions = positions;
    q.flags = flags;
    q.M = M;
    q.L = (int)L;
    q.N = (int)N;
    q.Np = (int)Np;
    q.Lp = wp.Lp;
    q.ut_stride = wp.ut_stride;
    q.ushared = wp.ushared;
    q.owner_bytes = wp.owner;
    void* args[] = {&q};
    ffsh::prof_begin(stream);
    cudaError_t e = cudaLaunchKernel(wp.fn, dim3(wp.grid), dim3(32 * wp.warps), args, wp.smem, stream);
    if (e != cudaSuccess) return fail(FFS_ECUDA, "launch failed: %s", cudaGetErrorString(e));
    ffsh::prof_end(stream);
    ++ffsh::launches();
    ffsh::clear_error();
    return FFS_OK;
  }
  HkpvPlan h;
  if (int rc = hkpv_plan(L, N, Np, dtype, M, h)) return rc;
  if (!ws || ws_bytes < h.total) return fail(FFS_ENOWS, "workspace %zu bytes < required %zu", ws_bytes, h.total);
  if (((uintptr_t)ws & (kAlign - 1)) != 0) return fail(FFS_EINVAL, "workspace not 256-byte aligned");
  const std::vector<int64_t> key = {2, (int64_t)(uintptr_t)U, L, N, dtype, M, Np, (int64_t)(uintptr_t)uniforms,
                                    (int64_t)(uintptr_t)positions, (int64_t)(uintptr_t)flags, (int64_t)(uintptr_t)ws};
  int rc = run_graph(key, stream, [&](cudaStream_t s) {
    return issue_hkpv(h, U, L, N, dtype, M, Np, uniforms, positions, flags, ws, s);
  });
  if (rc != FFS_OK) return rc;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(FFS_ECUDA, "CUDA error: %s", cudaGetErrorString(e));
  ffsh::clear_error();
  return FFS_OK;
}
}  // namespace

// ====================================================================== extern "C"
extern "C" {

size_t ffs_workspace_bytes(int64_t L, int64_t N, int64_t Nprime, ffs_dtype dtype, int64_t M) {
  return workspace_bytes(L, N, Nprime, dtype, M);
}

int ffs_sample(const void* U, int64_t L, int64_t N, ffs_dtype dtype, int64_t M, const double* uniforms,
               int32_t* positions, int32_t* sample_flags, void* workspace, size_t ws_bytes, void* stream) {
  return launch(U, L, N, dtype, M, N, uniforms, positions, sample_flags, workspace, ws_bytes,
                static_cast<cudaStream_t>(stream), 0, 0, nullptr);
}

int ffs_sample_marginal(const void* U, int64_t L, int64_t N, ffs_dtype dtype, int64_t M, int64_t Nprime,
                        const double* uniforms, int32_t* positions, int32_t* sample_flags, void* workspace,
                        size_t ws_bytes, void* stream) {
  return launch(U, L, N, dtype, M, Nprime, uniforms, positions, sample_flags, workspace, ws_bytes,
                static_cast<cudaStream_t>(stream), 0, 0, nullptr);
}

int ffs_debug_trace(const void* U, int64_t L, int64_t N, ffs_dtype dtype, int64_t M, int64_t Nprime,
                    const double* uniforms, int32_t* positions, int32_t* sample_flags, void* workspace,
                    size_t ws_bytes, void* stream, int64_t S0, int64_t S, double* weights) {
  if (S < 0 || S0 < 0 || (M > 0 && S0 + S > M))
    return fail(FFS_EINVAL, "trace range [%lld, %lld) outside [0, M=%lld)", (long long)S0, (long long)(S0 + S), (long long)M);
  return launch(U, L, N, dtype, M, Nprime, uniforms, positions, sample_flags, workspace, ws_bytes,
                static_cast<cudaStream_t>(stream), S0, S, weights);
}

// ---------------------------------------------------------------- host-buffer path
// Device layout inside the caller's workspace: [U | uniforms chunk x2 | positions chunk x2 |
// flags chunk x2 | sampling workspace]. Chunks alternate between two buffers so the copies of
// chunk c+1 overlap the kernel of chunk c.
namespace {
struct HostLayout {
  size_t u, uni[2], pos[2], flg[2], ws, total;
  int64_t chunk;
};
int64_t host_chunk(int64_t M) { return std::max<int64_t>(1, std::min<int64_t>(M, M > 32768 ? 16384 : M)); }
bool host_layout(int64_t L, int64_t N, int64_t Np, ffs_dtype dtype, int64_t M, HostLayout& h) {
  const size_t es = dtype == FFS_C128 ? 16 : 8;
  h.chunk = host_chunk(M);
  size_t o = 0;
  h.u = o; o = align_up(o + (size_t)L * N * es);
  for (int b = 0; b < 2; ++b) { h.uni[b] = o; o = align_up(o + (size_t)h.chunk * 2 * Np * 8); }
  for (int b = 0; b < 2; ++b) { h.pos[b] = o; o = align_up(o + (size_t)h.chunk * Np * 4); }
  for (int b = 0; b < 2; ++b) { h.flg[b] = o; o = align_up(o + (size_t)h.chunk * 4); }
  h.ws = o;
  const size_t need = workspace_bytes(L, N, Np, dtype, h.chunk);
  if (need == 0) return false;
  o += need;
  h.total = o;
  return true;
}

// Three-stage pipeline over sample chunks, double-buffered in the workspace: copy-in stream
// (U once, then uniforms of chunk c) -> caller's stream (sampling of chunk c) -> copy-out stream
// (positions/flags of chunk c). Streams/events are created once per host thread.
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

size_t ffs_host_workspace_bytes(int64_t L, int64_t N, int64_t Nprime, ffs_dtype dtype, int64_t M) {
  HostLayout h;
  if (!host_layout(L, N, Nprime, dtype, std::max<int64_t>(M, 1), h)) return 0;
  return h.total;
}

int ffs_sample_host(const void* U, int64_t L, int64_t N, ffs_dtype dtype, int64_t M, int64_t Nprime,
                    const double* uniforms, int32_t* positions, int32_t* sample_flags, void* workspace,
                    size_t ws_bytes, void* stream) {
  if (M == 0) return FFS_OK;
  if (int rc = check_shape(L, N, Nprime, dtype, M, true)) return rc;
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
                    h.total - h.ws, s0, 0, 0, nullptr);
    if (rc != FFS_OK) return rc;
    launches += ffsh::launches();
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
  ffsh::launches() = launches;
  return FFS_OK;
}

size_t ffs_lensemble_workspace_bytes(int64_t L, int64_t K, ffs_dtype dtype, int64_t M) {
  LensLayout y;
  return lens_layout(L, K, dtype, M, y) == FFS_OK ? y.total : 0;
}

int ffs_sample_lensemble(const void* V, const double* lambda, int64_t L, int64_t K, ffs_dtype dtype, int64_t M,
                         const double* uniforms, int32_t* positions, int32_t* counts, int32_t* sample_flags,
                         void* workspace, size_t ws_bytes, void* stream) {
  return launch_lensemble(V, lambda, L, K, dtype, M, uniforms, positions, counts, sample_flags, workspace, ws_bytes,
                          static_cast<cudaStream_t>(stream));
}

// ---------------------------------------------------------------- observables (ffs_observe.cuh)
static int obs_grid(int64_t work_items, int per_cta) {
  const int sms = ffsh::sm_count(ffsh::device());
  return (int)std::max<int64_t>(1, std::min<int64_t>((work_items + per_cta - 1) / per_cta, (int64_t)sms * 8));
}

int ffs_occupation(const int32_t* positions, int64_t M, int64_t Nprime, int64_t L, unsigned long long* occ,
                   void* stream) {
  ffsh::launches() = 0;
  if (M < 0 || Nprime < 1 || L < 1 || L > INT32_MAX) return fail(FFS_EINVAL, "invalid shape M=%lld N'=%lld L=%lld",
                                                              (long long)M, (long long)Nprime, (long long)L);
  if (!occ || (M > 0 && !positions)) return fail(FFS_EINVAL, "null positions/occ");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (cudaMemsetAsync(occ, 0, (size_t)L * 8, s) != cudaSuccess) return fail(FFS_ECUDA, "memset failed");
  if (M == 0) return FFS_OK;
  const int64_t n = M * Nprime;
  const int grid = obs_grid(n, ffsk::kObsThreads * 16);
  const bool sm = L * 4 <= 48 * 1024 * 4;
  ffsh::prof_begin(s);
  if (sm) {
    if (int rc = ffsh::ensure_max_smem(reinterpret_cast<const void*>(&ffsk::ffs_occupation_kernel<true>))) return rc;
    ffsk::ffs_occupation_kernel<true><<<grid, ffsk::kObsThreads, (size_t)L * 4, s>>>(positions, n, (int)L, occ);
  } else {
    ffsk::ffs_occupation_kernel<false><<<grid, ffsk::kObsThreads, 0, s>>>(positions, n, (int)L, occ);
  }
  ffsh::prof_end(s);
  ++ffsh::launches();
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? FFS_OK : fail(FFS_ECUDA, "occupation kernel: %s", cudaGetErrorString(e));
}

int ffs_pair_occupation(const int32_t* positions, int64_t M, int64_t Nprime, int64_t W, unsigned long long* pair,
                        void* stream) {
  ffsh::launches() = 0;
  if (M < 0 || Nprime < 1 || Nprime > 8192 || W < 1 || W > 46340)
    return fail(FFS_EINVAL, "invalid shape M=%lld N'=%lld W=%lld", (long long)M, (long long)Nprime, (long long)W);
  if (!pair || (M > 0 && !positions)) return fail(FFS_EINVAL, "null positions/pair");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (cudaMemsetAsync(pair, 0, (size_t)W * W * 8, s) != cudaSuccess) return fail(FFS_ECUDA, "memset failed");
  if (M == 0) return FFS_OK;
  const int warps = ffsk::kObsThreads / 32;
  if (int rc = ffsh::ensure_max_smem(reinterpret_cast<const void*>(&ffsk::ffs_pair_kernel))) return rc;
  ffsh::prof_begin(s);
  ffsk::ffs_pair_kernel<<<obs_grid(M, warps), ffsk::kObsThreads, (size_t)warps * Nprime * 4, s>>>(positions, M, (int)Nprime,
                                                                                               (int)W, pair);
  ffsh::prof_end(s);
  ++ffsh::launches();
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? FFS_OK : fail(FFS_ECUDA, "pair kernel: %s", cudaGetErrorString(e));
}

size_t ffs_gutzwiller_workspace_bytes(int64_t Nprime, int64_t L) {
  if (Nprime < 1 || L < 1 || L > INT32_MAX) return 0;
  return align_up((size_t)(Nprime + 1) * 8) + align_up((size_t)(Nprime + 1) * L * 8);
}

int ffs_gutzwiller_reweight(const int32_t* positions, int64_t Ms, int64_t Nprime, int64_t L, double V, double* result,
                            unsigned long long* dcount, void* workspace, size_t ws_bytes, void* stream) {
  ffsh::launches() = 0;
  if (Ms < 1 || Nprime < 1 || L < 1 || L > INT32_MAX || !std::isfinite(V))
    return fail(FFS_EINVAL, "invalid arguments Ms=%lld N'=%lld L=%lld", (long long)Ms, (long long)Nprime, (long long)L);
  if (!positions || !result) return fail(FFS_EINVAL, "null positions/result");
  const size_t need = ffs_gutzwiller_workspace_bytes(Nprime, L);
  if (!workspace || ws_bytes < need) return fail(FFS_ENOWS, "workspace %zu bytes < required %zu", ws_bytes, need);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  unsigned long long* dc = static_cast<unsigned long long*>(workspace);
  unsigned long long* od = reinterpret_cast<unsigned long long*>(static_cast<char*>(workspace) +
                                                                 align_up((size_t)(Nprime + 1) * 8));
  if (cudaMemsetAsync(workspace, 0, need, s) != cudaSuccess) return fail(FFS_ECUDA, "memset failed");
  const int warps = ffsk::kObsThreads / 32;
  const size_t smem = (size_t)warps * ((L + 31) / 32) * 4;
  if (smem > kMaxSmem) return fail(FFS_EINVAL, "L=%lld too large for the per-warp site bitmap", (long long)L);
  if (int rc = ffsh::ensure_max_smem(reinterpret_cast<const void*>(&ffsk::ffs_gutzwiller_kernel))) return rc;
  ffsh::prof_begin(s);
  ffsk::ffs_gutzwiller_kernel<<<obs_grid(Ms, warps), ffsk::kObsThreads, smem, s>>>(positions, Ms, (int)Nprime, (int)L,
                                                                                  dc, od);
  ffsk::ffs_reweight_finalize_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((L + 255) / 256, 1024)), 256, 0, s>>>(
      dc, od, (int)Nprime, (int)L, Ms, V, result);
  ffsh::prof_end(s);
  ffsh::launches() += 2;
  if (dcount && cudaMemcpyAsync(dcount, dc, (size_t)(Nprime + 1) * 8, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return fail(FFS_ECUDA, "dcount copy failed");
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? FFS_OK : fail(FFS_ECUDA, "gutzwiller kernels: %s", cudaGetErrorString(e));
}

size_t ffs_metropolis_workspace_bytes(int64_t L, int64_t N, int64_t Nprime, int64_t Mcond, ffs_dtype dtype, int64_t M) {
  MetroLayout y;
  return metro_layout(L, N, Nprime, Mcond, dtype, M, y) == FFS_OK ? y.total : 0;
}

int ffs_sample_metropolis(const void* U, int64_t L, int64_t N, ffs_dtype dtype, int64_t M, int64_t Nprime,
                          int64_t Mcond, const double* uniforms, int32_t* positions, int32_t* sample_flags,
                          void* workspace, size_t ws_bytes, void* stream) {
  return launch_metropolis(U, L, N, dtype, M, Nprime, Mcond, uniforms, positions, sample_flags, workspace, ws_bytes,
                           static_cast<cudaStream_t>(stream));
}

size_t ffs_hkpv_workspace_bytes(int64_t L, int64_t N, int64_t Nprime, ffs_dtype dtype, int64_t M) {
  HkpvPlan h;
  return hkpv_plan(L, N, Nprime, dtype, M, h) == FFS_OK ? h.total : 0;
}

int ffs_sample_hkpv(const void* U, int64_t L, int64_t N, ffs_dtype dtype, int64_t M, int64_t Nprime,
                    const double* uniforms, int32_t* positions, int32_t* sample_flags, void* workspace,
                    size_t ws_bytes, void* stream) {
  return launch_hkpv(U, L, N, dtype, M, Nprime, uniforms, positions, sample_flags, workspace, ws_bytes,
                     static_cast<cudaStream_t>(stream));
}

int ffs_last_launch_count(void) { return ffsh::launches(); }

int ffs_profile_enable(int on) {
  ffsh::g_prof = on != 0;
  ffsh::g_ev_pending = false;
  return FFS_OK;
}

float ffs_last_kernel_ms(void) {
  if (!ffsh::g_ev_pending) return -1.0f;
  float ms = -1.0f;
  if (cudaEventSynchronize(ffsh::g_ev1) != cudaSuccess) return -1.0f;
  if (cudaEventElapsedTime(&ms, ffsh::g_ev0, ffsh::g_ev1) != cudaSuccess) return -1.0f;
  return ms;
}

int ffs_set_option(int opt, double value) {
  if (opt <= 0 || opt >= ffsh::kNumOpts || opt > FFS_OPT_LAST) return fail(FFS_EINVAL, "unknown option %d", opt);
  auto& o = ffsh::opts();
  o.v[opt].store(std::isnan(value) || value < -1e300 ? ffsh::default_option(opt) : value);
  o.version.fetch_add(1);
  return FFS_OK;
}

double ffs_get_option(int opt) {
  if (opt <= 0 || opt >= ffsh::kNumOpts || opt > FFS_OPT_LAST) return NAN;
  return ffsh::option(opt);
}

int ffs_gram_counters(unsigned long long out[2], int reset) {
  ffsh::clear_error();
  if (!out) return fail(FFS_EINVAL, "null out");
  if (cudaMemcpyFromSymbol(out, ffsk::g_gram_stats, 2 * sizeof(unsigned long long)) != cudaSuccess)
    return fail(FFS_ECUDA, "cudaMemcpyFromSymbol failed");
  if (reset) {
    const unsigned long long z[2] = {0, 0};
    if (cudaMemcpyToSymbol(ffsk::g_gram_stats, z, sizeof(z)) != cudaSuccess) return fail(FFS_ECUDA, "cudaMemcpyToSymbol failed");
  }
  return FFS_OK;
}

const char* ffs_last_error(void) { return ffsh::g_err; }

}  // extern "C"
