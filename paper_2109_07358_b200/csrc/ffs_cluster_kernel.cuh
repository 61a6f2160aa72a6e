// Cluster-owner FFS kernel for large L (the C4 2D lattice and the C5 DPP-shaped workloads).
//
// Same mathematics as ffs_kernel.cuh (blocked left-looking randomized-pivot LU),
// but one sample is owned by a thread-block CLUSTER of CS CTAs (one per SM): CTA `rank` holds
// rows [rank*Lc, (rank+1)*Lc) of the L x B panel in registers (Lc = threads * R). The panel
// width B -- the reuse factor of every V element gathered from U in the contraction a3 -- is
// therefore bounded by the register files of CS SMs instead of one, which is what makes the
// contraction compute-bound for L = 4096..16384.
// Per draw (a4): CTA-local weights / prefix / totals, then each CTA publishes its total and
// fallback candidates into every CTA's shared memory (DSMEM stores) and the cluster barrier
// makes them visible; every CTA derives the same crossing CTA; the crossing CTA finds x_k and
// pushes the pivot row to all CTAs (DSMEM) before the second cluster barrier.
// W = A^{-1} V[X, later columns] lives in global memory (per cluster); its Gauss-Jordan update
// after each block is split over the cluster's CTAs by column.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ffs_kernel.cuh"

namespace ffsk {

constexpr int kMaxCS = 16;

struct ClusterParams {
  const double* U;         // [L][N] row-major scalars (complex interleaved)
  const double* Ut;        // [N][Lpt] transposed, zero-padded (workspace)
  int L, N, Np, Lc, Lpt;   // Lc rows per CTA, Lpt = CS * Lc
  int64_t M;
  const double* uniforms;  // [M][2Np]
  int32_t* positions;      // [M][Np]
  int32_t* flags;
  double* wfull;           // per cluster [Np][Np] scalars
  int64_t S0, S;           // debug trace of samples S0 .. S0+S-1
  double* trace;           // [S][Np][L] or null
  // STEP mode (lockstep-dense path, ffs_dense.cuh): one block step k0 for the Sb samples
  // base .. base+Sb-1 (cluster c <-> sample base+c); the panel comes from P = U Y
  const double* Pd;        // [L][ldY] panels, sample s in columns s*B .. s*B+B-1
  int64_t ldY;
  double* rowg;            // [Sb][B*B + B] pivot rows and inverse pivots of this block (out)
  const int32_t* permg;    // [M][Np] permutation prefixes (ffs_permute_kernel)
  uint32_t* chosen_g;      // [Sb][Lpt/32] rows drawn so far (bit per row)
  int k0, Sb;
  int gather;              // STEP: 1 = contract the gathered columns of Ut (no GEMM for this block)
  int panel_out;           // STEP + gather: 1 = only write the contracted panel to Pd ([L][B] per sample);
                           // the draws follow in ffs_gram_kernel + ffs_gram_draw_kernel (ffs_gram.cuh)
  int64_t base;
};

constexpr int kKC = 64;        // rows of W (or columns of the new rows) staged per chunk

template <typename T, int B>
struct ClusterLayout {
  size_t perm, pos, usel, row, pinv, wb, vnew, red, xch, total;
  __host__ __device__ ClusterLayout(int N, int Np) {
    size_t o = 0;
    perm = o; o = align16(o + sizeof(int) * N);
    pos = o;  o = align16(o + sizeof(int) * Np);
    usel = o; o = align16(o + sizeof(double) * Np);
    row = o;  o = align16(o + sizeof(T) * B * B);
    pinv = o; o = align16(o + sizeof(T) * B);
    wb = o;   o = align16(o + sizeof(T) * (size_t)kKC * B);  // chunk of Wb rows / new-row columns
    vnew = o; o = align16(o + sizeof(T) * (size_t)kKC * B);
    red = o;  o = align16(o + sizeof(double) * 64 + sizeof(int) * 96);
    xch = o;  o = align16(o + sizeof(double) * 4 * kMaxCS + 2 * sizeof(T) * B + 64);  // cluster exchange
    total = o;
  }
};

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cluster_size() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cluster_id_x() {
  unsigned r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned nclusters_x() {
  unsigned r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// store to the same shared-memory variable in CTA `rank` of this cluster
__device__ __forceinline__ void st_remote_f64(void* local_ptr, unsigned rank, double v) {
  unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(local_ptr)), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
}
__device__ __forceinline__ void st_remote_s32(void* local_ptr, unsigned rank, int v) {
  unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(local_ptr)), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(ra), "r"(v) : "memory");
}

// R consecutive rows of one U^T column (row0 and Lpt are multiples of R): 32-byte loads where they fit
template <typename T, int R>
__device__ __forceinline__ void ldrows(const T* __restrict__ base, T (&v)[R]) {
  constexpr int kD = sizeof(T) / 8 * R;  // doubles
  if constexpr (kD % 4 == 0 && (sizeof(T) == 8 ? R % 4 == 0 : R % 2 == 0)) {
    double* d = reinterpret_cast<double*>(&v[0]);
    const double* b = reinterpret_cast<const double*>(base);
#pragma unroll
    for (int q = 0; q < kD / 4; ++q)
      asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
          : "=d"(d[4 * q]), "=d"(d[4 * q + 1]), "=d"(d[4 * q + 2]), "=d"(d[4 * q + 3])
          : "l"(b + 4 * q));
  } else {
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = base[r];
  }
}

template <typename T, int R, int B, int MAXT, bool STEP = false>
__global__ void __launch_bounds__(MAXT, 1) ffs_cluster_kernel(const ClusterParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  using S = Sc<T>;
  constexpr int kD = S::kDoubles;
  const int t = threadIdx.x;
  const int lane = t & 31, warp = t >> 5;
  const int nw = blockDim.x >> 5;
  const unsigned rank = cluster_rank();
  const unsigned CS = cluster_size();
  const int L = p.L, N = p.N, Np = p.Np, Lc = p.Lc;
  const int row0 = (int)rank * Lc + t * R;  // first global row of this thread

  const ClusterLayout<T, B> lay(N, Np);
  int* perm = reinterpret_cast<int*>(smem + lay.perm);
  int* pos = reinterpret_cast<int*>(smem + lay.pos);
  double* usel = reinterpret_cast<double*>(smem + lay.usel);
  T* Row = reinterpret_cast<T*>(smem + lay.row);
  T* Pinv = reinterpret_cast<T*>(smem + lay.pinv);
  T* Wb = reinterpret_cast<T*>(smem + lay.wb);
  T* Vnew = reinterpret_cast<T*>(smem + lay.vnew);
  double* red = reinterpret_cast<double*>(smem + lay.red);
  int* redi = reinterpret_cast<int*>(smem + lay.red + sizeof(double) * 64);
  double* xtot = reinterpret_cast<double*>(smem + lay.xch);  // [CS] CTA totals
  int* xlast = reinterpret_cast<int*>(xtot + kMaxCS);        // [CS] last positive row (global) or -1
  int* xfree = xlast + kMaxCS;                                 // [CS] first unchosen row or INT_MAX
  int* xsel = xfree + kMaxCS;                                  // selected row (global)
  T* xrow = reinterpret_cast<T*>(reinterpret_cast<unsigned char*>(xsel) + 16);  // [B] pivot row
  T* xstage = xrow + B;                                        // [B] claimer's row (local)

  const int64_t cid = cluster_id_x();
  const int64_t ncl = nclusters_x();
  const T* Ug = reinterpret_cast<const T*>(p.U);
  const T* Utg = reinterpret_cast<const T*>(p.Ut);
  constexpr int kNone = 0x7fffffff;
  constexpr int kUnset = -0x7fffffff;  // xsel before the crossing CTA's push

  const int64_t nloc = STEP ? (int64_t)p.Sb : p.M;
  for (int64_t sl = cid; sl < nloc; sl += ncl) {
    const int64_t i = STEP ? p.base + sl : sl;
    // W = A^{-1} V[X, later columns]: per cluster, or per batch sample in STEP mode (it persists
    // across the block-step launches)
    T* Wf = reinterpret_cast<T*>(p.wfull) + (STEP ? sl : cid) * (int64_t)Np * Np;
    const double* urow = p.uniforms + i * 2 * (int64_t)Np;
    // ---- a1 permutation (every CTA computes the same one; STEP: precomputed prefix, and only the
    // entries this block step reads: the gathered columns m_0 .. m_{k0+B-1} when it contracts
    // them itself, and its own B selection uniforms)
    if constexpr (STEP) {
      const int kend = min(Np, p.k0 + B);
      if (p.gather)
        for (int j = t; j < kend; j += blockDim.x) perm[j] = p.permg[i * Np + j];
      for (int j = p.k0 + t; j < kend; j += blockDim.x) usel[j] = urow[Np + j];
    } else {
      for (int j = t; j < N; j += blockDim.x) perm[j] = j;
      for (int j = t; j < Np; j += blockDim.x) usel[j] = urow[Np + j];
    }
    __syncthreads();
    if (!STEP && t == 0) {
      for (int j = 0; j < Np; ++j) {
        const int n = N - j;
        int r = (int)floor(urow[j] * (double)n);
        r = (r > n - 1 ? n - 1 : r) + j;
        const int a = perm[j];
        perm[j] = perm[r];
        perm[r] = a;
      }
    }
    __syncthreads();
    uint32_t chosen = 0;
    int flag = 0;
    uint32_t* chw = nullptr;  // STEP: this thread's word of the drawn-row bitmap
    if constexpr (STEP) {
      static_assert(32 % R == 0, "a thread's rows share one bitmap word");
      chw = p.chosen_g + sl * (int64_t)(p.Lpt / 32) + row0 / 32;
      chosen = (*chw >> (row0 & 31)) & ((1u << R) - 1u);
    }

    for (int k0 = STEP ? p.k0 : 0; k0 < Np; k0 += B) {
      const int nb = min(B, Np - k0);
      // ---- a3 panel for this CTA's rows (W in global memory is final for rows < k0 after the
      // previous block's update + cluster barrier; its rows are staged kKC at a time)
      T P[R][B];
      // STEP with p.gather: early blocks (small k0) contract the gathered columns here, like the
      // cluster path, instead of paying the dense GEMM's full-N contraction
      const bool from_gemm = STEP && !p.gather;
      if (from_gemm) {
        // the panel from the dense GEMM P = U Y, per-sample layout [L][B] (rows >= L are zero):
        // this thread's R rows are R*B contiguous scalars, read as 16-byte vectors
        const double2* pb = reinterpret_cast<const double2*>(reinterpret_cast<const T*>(p.Pd) +
                                                             ((size_t)sl * L + row0) * B);
        constexpr int kV = B * S::kDoubles / 2;  // 16-byte vectors per row
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const bool in = row0 + r < L;
#pragma unroll
          for (int v = 0; v < kV; ++v) {
            const double2 d2 = in ? pb[r * kV + v] : make_double2(0.0, 0.0);
            if constexpr (S::kDoubles == 1) {
              P[r][2 * v] = d2.x;
              P[r][2 * v + 1] = d2.y;
            } else {
              reinterpret_cast<double*>(&P[r][v])[0] = d2.x;
              reinterpret_cast<double*>(&P[r][v])[1] = d2.y;
            }
          }
          if (nb < B) {
#pragma unroll
            for (int c = 0; c < B; ++c)
              if (c >= nb) P[r][c] = S::zero();
          }
        }
      } else {
#pragma unroll
      for (int c = 0; c < B; ++c) {
        const T* base = Utg + (size_t)perm[min(k0 + c, Np - 1)] * p.Lpt + row0;
        T v[R];
        ldrows(base, v);
#pragma unroll
        for (int r = 0; r < R; ++r) P[r][c] = (c < nb) ? v[r] : S::zero();
      }
      }
      // contraction over the k0 earlier columns; W rows are staged kKC at a time in shared memory
      for (int c0 = 0; c0 < (from_gemm ? 0 : k0); c0 += kKC) {
        const int kc = min(kKC, k0 - c0);
        __syncthreads();
        for (int idx = t; idx < kc * B; idx += blockDim.x) {
          const int ii = idx / B, c = idx % B;
          Wb[idx] = c < nb ? Wf[(size_t)(c0 + ii) * Np + k0 + c] : S::zero();
        }
        __syncthreads();
#pragma unroll 2
        for (int i2 = 0; i2 < kc; ++i2) {
          const T* base = Utg + (size_t)perm[c0 + i2] * p.Lpt + row0;
          T v[R];
          ldrows(base, v);
          T wb[B];
#pragma unroll
          for (int c = 0; c < B; ++c) wb[c] = Wb[i2 * B + c];
#pragma unroll
          for (int c = 0; c < B; ++c)
#pragma unroll
            for (int r = 0; r < R; ++r) P[r][c] = S::fms(v[r], wb[c], P[r][c]);
        }
      }
      bool draws_here = true;
      if constexpr (STEP) {
        if (p.panel_out) {
          // the gathered panel goes to global memory in the GEMM's layout; no draws in this kernel
          double2* pb = reinterpret_cast<double2*>(const_cast<T*>(reinterpret_cast<const T*>(p.Pd)) + ((size_t)sl * L + row0) * B);
          constexpr int kV = B * S::kDoubles / 2;
#pragma unroll
          for (int r = 0; r < R; ++r)
            if (row0 + r < L) {
#pragma unroll
              for (int v = 0; v < kV; ++v) {
                if constexpr (S::kDoubles == 1) pb[r * kV + v] = make_double2(P[r][2 * v], P[r][2 * v + 1]);
                else pb[r * kV + v] = make_double2(reinterpret_cast<double*>(&P[r][v])[0], reinterpret_cast<double*>(&P[r][v])[1]);
              }
            }
          draws_here = false;
        }
      }
      // rows drawn earlier: exactly zero weight in the first column of this block
#pragma unroll
      for (int r = 0; r < R; ++r)
        if ((chosen >> r) & 1u) P[r][0] = S::zero();

      // ---- a4/a5: nb sequential draws. Per draw: CTA scan (one CTA barrier), each CTA's total
      // to every CTA (thread q -> CTA q), cluster barrier #1, every warp derives T, its CTA's
      // offset and the crossing CTA with CS lanes, the one warp of the crossing CTA whose range
      // holds u*T pushes x_k and the pivot row to every CTA, cluster barrier #2, rank-1 update.
      // The fallbacks of reading Q5 (T not finite/positive, no crossing because of rounding)
      // take an extra, cluster-uniform round (rare).
      static_for<0, B>([&](auto rrc) {
        constexpr int rr = decltype(rrc)::value;
        if (rr < nb && draws_here) {
          const int k = k0 + rr;
          double w[R], c[R];
          double acc = 0.0;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            w[r] = S::abs2(P[r][rr]);
            acc += w[r];
            c[r] = acc;
          }
          const double incl = warp_incl_scan(acc, lane);
          double* redp = red;  // warp totals
          if (lane == 31) redp[warp] = incl;
          __syncthreads();
          double woff, Tc;
          {
            const double wt = lane < nw ? redp[lane] : 0.0;
            const double ws = warp_incl_scan(wt, lane);
            woff = __shfl_sync(0xffffffffu, ws, warp > 0 ? warp - 1 : 0);
            woff = warp > 0 ? woff : 0.0;
            Tc = __shfl_sync(0xffffffffu, ws, 31);
          }
          double excl = __shfl_up_sync(0xffffffffu, incl, 1);
          excl = (lane == 0 ? 0.0 : excl) + woff;
          const double* xt = xtot;
          if (t < (int)CS) st_remote_f64(&xtot[rank], (unsigned)t, Tc);
          if (t == 0) *xsel = kUnset;  // remote pushes of this step arrive after barrier #1
          cluster_sync_all();  // #1: CTA totals visible
          // cluster-uniform T, this CTA's offset and the crossing CTA (lanes q < CS)
          const double u = usel[k];
          double Ttot, off;
          int owner_cta;
          {
            const double tq = lane < (int)CS ? xt[lane] : 0.0;
            double ci = tq;
#pragma unroll
            for (int d = 1; d < kMaxCS; d <<= 1) {
              const double y = __shfl_up_sync(0xffffffffu, ci, d);
              ci = lane >= d ? ci + y : ci;
            }
            Ttot = __shfl_sync(0xffffffffu, ci, kMaxCS - 1);
            double ce = __shfl_up_sync(0xffffffffu, ci, 1);  // exclusive prefix
            ce = lane == 0 ? 0.0 : ce;
            off = __shfl_sync(0xffffffffu, ce, (int)rank);
            const double thr0 = u * Ttot;
            const unsigned ob = __ballot_sync(0xffffffffu, lane < (int)CS && tq > 0.0 && ci > thr0);
            owner_cta = ob ? __ffs(ob) - 1 : -1;
          }
          const bool ok = (Ttot > 0.0) && (Ttot <= 1.7976931348623157e308);
          const double thr = u * Ttot;
          if (ok && owner_cta == (int)rank) {
            const double thl = thr - off;
            const double wt = redp[warp];
            // exactly one warp is responsible for the threshold (the first / last absorb rounding)
            const bool mine = (warp == 0 || thl >= woff) && (warp == nw - 1 || thl - woff < wt);
            const double tp = fmax(thl - excl, 0.0);
            int rs = R;
#pragma unroll
            for (int r = R - 1; r >= 0; --r)
              if (w[r] > 0.0 && c[r] > tp) rs = r;
            const unsigned bal = __ballot_sync(0xffffffffu, mine && rs < R);
            if (bal != 0u) {
              const int ln = __ffs(bal) - 1;
              const int rsel = __shfl_sync(0xffffffffu, rs, ln);
              const int xs = (int)rank * Lc + (warp * 32 + ln) * R + rsel;
              // the claiming lane's row by a select tree (constant register indices)
#pragma unroll
              for (int cc = 0; cc < B; ++cc) {
                T tr[R];
#pragma unroll
                for (int r = 0; r < R; ++r) tr[r] = P[r][cc];
#pragma unroll
                for (int wd = 1; wd < R; wd <<= 1)
#pragma unroll
                  for (int q = 0; q < R; q += 2 * wd) tr[q] = (rsel & wd) ? tr[q + wd] : tr[q];
                if (lane == ln) xstage[cc] = tr[0];
              }
              __syncwarp();
              const double* xs_src = reinterpret_cast<const double*>(xstage);
              double* xr_dst = reinterpret_cast<double*>(xrow);
              for (int idx = lane; idx < (int)CS * B * kD; idx += 32) {
                const int q = idx / (B * kD), e = idx % (B * kD);
                st_remote_f64(xr_dst + e, (unsigned)q, xs_src[e]);
              }
              if (lane < (int)CS) st_remote_s32(xsel, (unsigned)lane, xs);
              if (lane == ln) chosen |= 1u << rsel;
            }
          }
          if (p.trace != nullptr && (uint64_t)(i - p.S0) < (uint64_t)p.S) {
            const double inv = Ttot > 0.0 ? 1.0 / Ttot : 0.0;
            double* tr = p.trace + ((i - p.S0) * Np + k) * (int64_t)L;
#pragma unroll
            for (int r = 0; r < R; ++r)
              if (row0 + r < L) tr[row0 + r] = w[r] * inv;
          }
          cluster_sync_all();  // #2: x_k and the pivot row visible in every CTA
          int xsel_k = *xsel;
          const T* xr = xrow;
          if (xsel_k == kUnset) {
            // rare (cluster-uniform): T not finite/positive -> smallest unchosen row (flag bit0);
            // no crossing -> the crossing CTA's (or, without one, the cluster's) last positive row
            if (!ok) flag |= 1;
            int rl = -1, rf = kNone;
#pragma unroll
            for (int r = R - 1; r >= 0; --r)
              if (row0 + r < L && !((chosen >> r) & 1u)) rf = row0 + r;
#pragma unroll
            for (int r = 0; r < R; ++r)
              if (w[r] > 0.0) rl = row0 + r;
            const int wl = __reduce_max_sync(0xffffffffu, rl);
            const int wf = __reduce_min_sync(0xffffffffu, rf);
            if (lane == 0) {
              redi[warp] = wl;
              redi[32 + warp] = wf;
            }
            __syncthreads();
            if (t < (int)CS) {
              int cl = -1, cf = kNone;
              for (int q = 0; q < nw; ++q) {
                cl = max(cl, redi[q]);
                cf = min(cf, redi[32 + q]);
              }
              st_remote_s32(&xlast[rank], (unsigned)t, cl);
              st_remote_s32(&xfree[rank], (unsigned)t, cf);
            }
            cluster_sync_all();
            int fb_last = -1, fb_free = kNone;
            for (unsigned q = 0; q < CS; ++q) {
              fb_last = max(fb_last, xlast[q]);
              fb_free = min(fb_free, xfree[q]);
            }
            const int xs = !ok ? fb_free : (owner_cta >= 0 ? xlast[owner_cta] : fb_last);
            if ((unsigned)(xs / Lc) == rank) {  // the holder thread pushes (serially; rare)
              const int own = (xs - (int)rank * Lc) / R, orow = (xs - (int)rank * Lc) % R;
#pragma unroll
              for (int cc = 0; cc < B; ++cc) {
                T tr[R];
#pragma unroll
                for (int r = 0; r < R; ++r) tr[r] = P[r][cc];
#pragma unroll
                for (int wd = 1; wd < R; wd <<= 1)
#pragma unroll
                  for (int q = 0; q < R; q += 2 * wd) tr[q] = (orow & wd) ? tr[q + wd] : tr[q];
                if (t == own) {
                  const double* src = reinterpret_cast<const double*>(&tr[0]);
                  double* dst = reinterpret_cast<double*>(&xrow[cc]);
                  for (unsigned q = 0; q < CS; ++q)
#pragma unroll
                    for (int h = 0; h < kD; ++h) st_remote_f64(dst + h, q, src[h]);
                }
              }
              if (t == own) {
                for (unsigned q = 0; q < CS; ++q) st_remote_s32(xsel, q, xs);
                chosen |= 1u << orow;
              }
            }
            cluster_sync_all();
            xsel_k = *xsel;
            xr = xrow;
          }
          FFS_CHECK(xsel_k >= 0 && xsel_k < L);
          if (t == 0) pos[k] = xsel_k;
          if (t < B) Row[rr * B + t] = xr[t];
          const T piv = xr[rr];
          if (S::abs2(piv) < 1e-12 * Ttot) flag |= 2;
          const T ip = S::recip(piv);
          if (t == 0) Pinv[rr] = ip;
          // rank-1 update of the remaining panel columns; drawn rows get exactly zero in the
          // next draw's column (the only column whose weights are formed)
          T lmul[R];
#pragma unroll
          for (int r = 0; r < R; ++r) lmul[r] = S::mul(P[r][rr], ip);
#pragma unroll
          for (int cc = rr + 1; cc < B; ++cc) {
            const T pc = xr[cc];
#pragma unroll
            for (int r = 0; r < R; ++r)
              P[r][cc] = (cc == rr + 1 && ((chosen >> r) & 1u)) ? S::zero() : S::fms(lmul[r], pc, P[r][cc]);
          }
        }
      });

      // ---- Gauss-Jordan update of W with the nb new rows, columns split over the cluster
      // (thread <-> one later column j; the new rows' entries in columns < k0 and W's rows < k0
      // are staged kKC at a time through shared memory)
      if constexpr (STEP) {
        // the Gauss-Jordan update runs batched in ffs_dense_gj_kernel: hand it S = L U of this block
        __syncthreads();  // the last draw's Row / Pinv entries come from other warps
        if (draws_here && rank == 0 && t < B * B + B) {
          T* rg = reinterpret_cast<T*>(p.rowg) + sl * (B * B + B);
          rg[t] = t < B * B ? Row[t] : Pinv[t - B * B];
        }
      }
      if (!STEP && k0 + nb < Np) {
       __syncthreads();  // Row / Pinv / pos of the block's last draw come from other warps
       for (int jt = k0 + nb; jt < Np; jt += (int)CS * blockDim.x) {  // column tiles (uniform trip count)
        const int j = jt + (int)rank * blockDim.x + t;
        const bool has = j < Np;
        T z[B];
#pragma unroll
        for (int tt = 0; tt < B; ++tt)
          z[tt] = (has && tt < nb) ? Ug[(size_t)pos[k0 + tt] * N + perm[j]] : S::zero();
        // R_new[:, j] = V[X_new, j] - V[X_new, 0:k0] W[0:k0, j]
        for (int c0 = 0; c0 < k0; c0 += kKC) {
          const int kc = min(kKC, k0 - c0);
          __syncthreads();
          for (int idx = t; idx < kc * B; idx += blockDim.x) {
            const int ii = idx / B, tt = idx % B;
            Vnew[idx] = tt < nb ? Ug[(size_t)pos[k0 + tt] * N + perm[c0 + ii]] : S::zero();
          }
          __syncthreads();
          if (has) {
            int ii = 0;
            for (; ii + 8 <= kc; ii += 8) {
              T w8[8];
#pragma unroll
              for (int uu = 0; uu < 8; ++uu) w8[uu] = Wf[(size_t)(c0 + ii + uu) * Np + j];
#pragma unroll
              for (int uu = 0; uu < 8; ++uu)
#pragma unroll
                for (int tt = 0; tt < B; ++tt) z[tt] = S::fms(Vnew[(ii + uu) * B + tt], w8[uu], z[tt]);
            }
            for (; ii < kc; ++ii) {
              const T wij = Wf[(size_t)(c0 + ii) * Np + j];
#pragma unroll
              for (int tt = 0; tt < B; ++tt) z[tt] = S::fms(Vnew[ii * B + tt], wij, z[tt]);
            }
          }
        }
        if (has) {
#pragma unroll
          for (int tt = 1; tt < B; ++tt)
            if (tt < nb) {
#pragma unroll
              for (int s2 = 0; s2 < tt; ++s2) z[tt] = S::fms(S::mul(Row[tt * B + s2], Pinv[s2]), z[s2], z[tt]);
            }
#pragma unroll
          for (int tt = B - 1; tt >= 0; --tt)
            if (tt < nb) {
#pragma unroll
              for (int s2 = tt + 1; s2 < B; ++s2)
                if (s2 < nb) z[tt] = S::fms(Row[tt * B + s2], z[s2], z[tt]);
              z[tt] = S::mul(z[tt], Pinv[tt]);
            }
#pragma unroll
          for (int tt = 0; tt < B; ++tt)
            if (tt < nb) Wf[(size_t)(k0 + tt) * Np + j] = z[tt];
        }
        // W[0:k0, j] -= Wb Z[:, j]
        for (int c0 = 0; c0 < k0; c0 += kKC) {
          const int kc = min(kKC, k0 - c0);
          __syncthreads();
          for (int idx = t; idx < kc * B; idx += blockDim.x) {
            const int ii = idx / B, c = idx % B;
            Wb[idx] = c < nb ? Wf[(size_t)(c0 + ii) * Np + k0 + c] : S::zero();
          }
          __syncthreads();
          if (has) {
            int ii = 0;
            for (; ii + 8 <= kc; ii += 8) {
              T a8[8];
#pragma unroll
              for (int uu = 0; uu < 8; ++uu) a8[uu] = Wf[(size_t)(c0 + ii + uu) * Np + j];
#pragma unroll
              for (int uu = 0; uu < 8; ++uu) {
#pragma unroll
                for (int tt = 0; tt < B; ++tt) a8[uu] = S::fms(Wb[(ii + uu) * B + tt], z[tt], a8[uu]);
                Wf[(size_t)(c0 + ii + uu) * Np + j] = a8[uu];
              }
            }
            for (; ii < kc; ++ii) {
              T a = Wf[(size_t)(c0 + ii) * Np + j];
#pragma unroll
              for (int tt = 0; tt < B; ++tt) a = S::fms(Wb[ii * B + tt], z[tt], a);
              Wf[(size_t)(c0 + ii) * Np + j] = a;
            }
          }
        }
       }
        __threadfence();
        cluster_sync_all();  // W visible to every CTA before the next block's Wb load
      }
      if constexpr (STEP) break;
    }
    // ---- a6: positions (rank 0) and flags (OR over the cluster, collected in rank 0)
    const int fcta = (__syncthreads_or(flag & 1) ? 1 : 0) | (__syncthreads_or(flag & 2) ? 2 : 0);
    if constexpr (STEP) {
      if (p.panel_out) continue;  // no draws here: nothing to publish, no DSMEM traffic to fence
      const int nbs = min(B, Np - p.k0);
      if (rank == 0)
        for (int j = p.k0 + t; j < p.k0 + nbs; j += blockDim.x) p.positions[i * Np + j] = pos[j];
      const uint32_t mine = chosen << (row0 & 31);
      if (mine) atomicOr(chw, mine);
      if (t == 0 && fcta != 0 && p.flags != nullptr) atomicOr(reinterpret_cast<unsigned*>(p.flags + i), (unsigned)fcta);
      cluster_sync_all();  // no CTA starts the next sample while DSMEM traffic of this one is pending
      continue;
    }
    if (rank == 0)
      for (int j = t; j < Np; j += blockDim.x) p.positions[i * Np + j] = pos[j];
    if (t == 0) st_remote_s32(&xfree[rank], 0, fcta);
    cluster_sync_all();
    if (rank == 0 && t == 0 && p.flags != nullptr) {
      int f = 0;
      for (unsigned q = 0; q < CS; ++q) f |= xfree[q];
      p.flags[i] = f;
    }
    cluster_sync_all();
  }
}

}  // namespace ffsk
