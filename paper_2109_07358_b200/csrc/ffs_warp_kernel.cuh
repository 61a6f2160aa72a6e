// Warp-owner FFS kernels for small real problems (L <= 32*R, N' <= kMaxNpWarp): the headline
// double-well workload (L=256, N=32) and the tiny exact-check config.
//
// Same mathematics as ffs_kernel.cuh (blocked left-looking randomized-pivot LU: panel
// contraction, B sequential draws on the register panel, Gauss-Jordan update of
// W = A^{-1} V[X, later cols]); organised for throughput on one SM (ffs_seg_kernel):
//   * one CTA per SM holds U^T once in shared memory (bank-conflict-free swizzle) and runs
//     independent sample owners: G-lane segments of its warps (G = 32 for C2: one sample per
//     warp; G = 4 for C1); everything a sample needs (W, pivot rows, new rows, permutation,
//     selection uniforms) lives in that owner's shared-memory slice;
//   * segment lane l owns rows l*R .. l*R+R-1 (index order == scan order); the L x B panel is in
//     registers;
//   * the draw of step r+1 (scan, crossing search) is issued before the rank-1 update of the
//     panel columns r+2.. so the shuffle latency overlaps FP64 work (one-column lookahead);
//   * the permutation rows come precomputed from ffs_permute_kernel.
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "ffs_kernel.cuh"

namespace ffsk {

constexpr int kMaxNpWarp = 48;

struct WarpLayout {
  size_t perm, pos, usel, row, pinv, wf, vnt, dump, total;
  int ldw;  // row stride of W: Np + B rounded to even; columns [Np, ldw) stay zero
  // seg: layout of the segmented kernel (no dump slice; W without padding columns when B | N')
  __host__ __device__ WarpLayout(int Np, int B, bool seg = false) {
    // (Np + 2 when B | N': rows of W start 16 bytes apart in bank space, so the flat
    // Gauss-Jordan mapping's (row, column) accesses do not collide)
    ldw = (seg && Np % B == 0) ? ((Np + 3) & ~1) : ((Np + B + 1) & ~1);
    size_t o = 0;
    perm = o; o = align16(o + sizeof(int) * Np);
    pos = o;  o = align16(o + sizeof(int) * Np);
    usel = o; o = align16(o + sizeof(double) * Np);
    row = o;  o = align16(o + sizeof(double) * B * B);
    pinv = o; o = align16(o + sizeof(double) * B);
    wf = o;   o = align16(o + sizeof(double) * (size_t)Np * ldw);
    vnt = o;  o = align16(o + sizeof(double) * (size_t)Np * B);
    dump = o; o = align16(o + (seg ? 0 : sizeof(double) * 16 * 8));  // owner's R x B panel (legacy)
    total = o;
  }
};

struct WarpParams {
  const double* U;        // [L][N] row-major
  const int32_t* perm;    // [M][Np] from ffs_permute_kernel
  const double* uniforms; // [M][2Np]
  int32_t* positions;     // [M][Np]
  int32_t* flags;         // [M] or null
  int64_t M;
  int L, N, Np, Lp, ut_stride;
  size_t ushared, owner_bytes;
  int64_t S;
  double* trace;          // [S][Np][L] or null
  int dbg;                // development: bit0 skip GEMM, bit1 trivial draws, bit2 skip GJ (WRONG results),
                          // bit3 per-phase clock64 accounting into timing[0..7]
  unsigned long long* timing;
  double* wfull;          // producer/consumer kernel: per (pair, slot) W [N'][ldw] in global memory
};

// Result of the branch-free part of a draw.
struct Draw {
  unsigned ball;  // lanes whose inclusive prefix exceeds u*T (the crossing lane is the first)
  int rsel;       // in the crossing lane: the first row with C(x) > u*T
  double T;       // total weight
};

// U [L][N] -> per-sample permutation prefix [M][Np] (a1 rule, reading Q6); one thread per sample.
static __global__ void ffs_permute_kernel(const double* __restrict__ uniforms, int32_t* __restrict__ perm, int64_t M,
                                   int N, int Np) {
  extern __shared__ int pscratch[];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // per-thread working permutation, interleaved across the block ([N][blockDim]): the threads of
  // a warp touch 32 consecutive words (no bank conflicts)
  int* m = pscratch + threadIdx.x;
  const int bs = blockDim.x;
  if (i >= M) return;
  for (int j = 0; j < N; ++j) m[j * bs] = j;
  const double* u = uniforms + i * 2 * (int64_t)Np;
  for (int j = 0; j < Np; ++j) {
    const int n = N - j;
    int r = (int)floor(u[j] * (double)n);
    r = (r > n - 1 ? n - 1 : r) + j;
    const int a = m[j * bs];
    const int b = m[r * bs];
    m[r * bs] = a;
    perm[i * Np + j] = b;
  }
}

// =====================================================================================
// Segmented warp kernel: a warp is split into 32/G segments of G lanes, one sample per segment.
// Warp-wide instructions (scan levels, ballots, broadcasts, shared loads, the reciprocal of the
// pivot) then serve 32/G samples at once, and the register file holds 32/G panels per warp.
// Lane s of a segment owns rows s*R .. s*R+R-1 of its sample (index order = scan order).
// =====================================================================================
template <int G>
struct SegOps {
  // v + (value of segment lane - d) for segment lanes >= d
  __device__ __forceinline__ static double scan_level(double v, int d) {
    double y = __shfl_up_sync(0xffffffffu, v, d, G);
    y = ((int)(threadIdx.x & (G - 1)) >= d) ? y : 0.0;  // v >= 0: v + 0.0 == v
    return v + y;
  }
  // value of segment lane - 1, 0 for the first segment lane
  __device__ __forceinline__ static double prev(double v) {
    const double y = __shfl_up_sync(0xffffffffu, v, 1, G);
    return (threadIdx.x & (G - 1)) != 0 ? y : 0.0;
  }
  // value of the last lane of the segment
  __device__ __forceinline__ static double last(double v) { return __shfl_sync(0xffffffffu, v, G - 1, G); }
};

// Branch-free part of a draw for one segment: returns the crossing lanes of
// this lane's segment (bit i = segment lane i), the crossing row in this lane, and T.
// Whole-warp draw (G = 32, R <= 8) with a shorter dependency chain: the local inclusive prefix is
// kept (no second pass), and the 32-lane scan runs as a 3-level scan inside 8-lane groups plus
// the group offsets read from the group-final lanes (one shuffle round instead of two levels).
// Every prefix value compared against the threshold is computed exactly as the previous lane's
// inclusive value would be, so the crossing lane and row are consistent (reading Q5).
template <int R>
__device__ __forceinline__ Draw warp_draw_fast(const double (&col)[R], double u, int lane) {
  double c[R];
  c[0] = col[0] * col[0];
#pragma unroll
  for (int r = 1; r < R; ++r) c[r] = fma(col[r], col[r], c[r - 1]);
  const double tot = c[R - 1];
  double li = tot;
  li = SegOps<8>::scan_level(li, 1);
  li = SegOps<8>::scan_level(li, 2);
  li = SegOps<8>::scan_level(li, 4);
  const double le = SegOps<8>::prev(li);
  const double g0 = __shfl_sync(0xffffffffu, li, 7);
  const double g1 = __shfl_sync(0xffffffffu, li, 15);
  const double g2 = __shfl_sync(0xffffffffu, li, 23);
  const double g3 = __shfl_sync(0xffffffffu, li, 31);
  const double o1 = g0, o2 = o1 + g1, o3 = o2 + g2;
  Draw d;
  d.T = o3 + g3;
  const int grp = lane >> 3;
  const double off = grp == 0 ? 0.0 : (grp == 1 ? o1 : (grp == 2 ? o2 : o3));
  const double excl = off + le;
  const bool ok = (d.T > 0.0) && (d.T < INFINITY);
  const double tq = fma(u, d.T, -excl);
  const double tp = tq > 0.0 ? tq : 0.0;
  d.ball = __ballot_sync(0xffffffffu, ok && (tot > tp));
  unsigned m = 0;
#pragma unroll
  for (int r = 0; r < R - 1; ++r) m |= (c[r] <= tp) ? (1u << r) : 0u;
  d.rsel = __popc(m);
  return d;
}

template <int R, int G, bool KEEP = false>
__device__ __forceinline__ Draw seg_draw(const double (&col)[R], double u, int seg) {
  if constexpr (false && G == 32 && R <= 8) {  // measured slower (646 vs 544 cycles/draw)
    return warp_draw_fast<R>(col, u, threadIdx.x & 31);
  }
  if constexpr (KEEP && R <= 8) {
    // same partial sums as the two-pass form below (bit-identical), kept in registers so the
    // row search after the ballot is R-1 independent compares instead of a dependent FMA chain
    double cs[R];
    cs[0] = col[0] * col[0];
#pragma unroll
    for (int r = 1; r < R; ++r) cs[r] = fma(col[r], col[r], cs[r - 1]);
    const double tot = cs[R - 1];
    double incl = tot;
#pragma unroll
    for (int d = 1; d < G; d <<= 1) incl = SegOps<G>::scan_level(incl, d);
    const double excl = SegOps<G>::prev(incl);
    Draw d;
    d.T = SegOps<G>::last(incl);
    const bool ok = (d.T > 0.0) && (d.T <= 1.7976931348623157e308);  // positive and finite
    const double tq = fma(u, d.T, -excl);
    const double tp = tq > 0.0 ? tq : 0.0;
    const unsigned b = __ballot_sync(0xffffffffu, ok && (tot > tp));
    d.ball = (G == 32) ? b : ((b >> (seg * G)) & ((1u << G) - 1u));
    int cnt = 0;
#pragma unroll
    for (int r = 0; r < R - 1; ++r) cnt += (cs[r] <= tp) ? 1 : 0;
    d.rsel = cnt;
    return d;
  }
  // Pass 1: lane total of w_r = col_r^2 (index order; for R > 8 two parallel half chains).
  constexpr int H = R > 8 ? R / 2 : R;
  double h1 = col[0] * col[0];
#pragma unroll
  for (int r = 1; r < H; ++r) h1 = fma(col[r], col[r], h1);
  double tot = h1;
  double h2 = 0.0;
  if constexpr (R > 8) {
    h2 = col[H] * col[H];
#pragma unroll
    for (int r = H + 1; r < R; ++r) h2 = fma(col[r], col[r], h2);
    tot = h1 + h2;
  }
  double incl = tot;
#pragma unroll
  for (int d = 1; d < G; d <<= 1) incl = SegOps<G>::scan_level(incl, d);
  const double excl = SegOps<G>::prev(incl);
  Draw d;
  d.T = SegOps<G>::last(incl);
  const bool ok = (d.T > 0.0) && (d.T <= 1.7976931348623157e308);  // positive and finite
  // crossing threshold relative to this lane's exclusive prefix, clamped at 0 so that a lane
  // whose rounded prefix already passed u*T still lands on its first positive weight
  const double tq = fma(u, d.T, -excl);
  const double tp = tq > 0.0 ? tq : 0.0;
  const unsigned b = __ballot_sync(0xffffffffu, ok && (tot > tp));
  d.ball = (G == 32) ? b : ((b >> (seg * G)) & ((1u << G) - 1u));
  // Pass 2: the same partial sums again (bit-identical), count rows with C_r <= tp (r < R-1).
  unsigned m = 0;
  double a = col[0] * col[0];
  m |= (a <= tp) ? 1u : 0u;
#pragma unroll
  for (int r = 1; r < H && r < R - 1; ++r) {
    a = fma(col[r], col[r], a);
    m |= (a <= tp) ? (1u << r) : 0u;
  }
  if constexpr (R > 8) {
    double bb = col[H] * col[H];
    m |= (h1 + bb <= tp) ? (1u << H) : 0u;
#pragma unroll
    for (int r = H + 1; r < R - 1; ++r) {
      bb = fma(col[r], col[r], bb);
      m |= (h1 + bb <= tp) ? (1u << r) : 0u;
    }
  }
  d.rsel = __popc(m);
  return d;
}

// Rare paths for one segment; every lane of the warp calls it (segments may differ).
template <int R, int G>
__device__ __noinline__ int seg_fallback(const double* col, double T, uint32_t chosen, int L, int sl, int seg) {
  const bool ok = (T > 0.0) && isfinite(T);
  int rl = -1, rf = R;
  for (int r = 0; r < R; ++r) {
    if (col[r] * col[r] > 0.0) rl = r;
    if (rf == R && sl * R + r < L && !((chosen >> r) & 1u)) rf = r;
  }
  const unsigned mseg = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (seg * G));
  const unsigned bl = __ballot_sync(0xffffffffu, rl >= 0) & mseg;
  const unsigned bf = __ballot_sync(0xffffffffu, rf < R) & mseg;
  int ln, rr;
  if (ok && bl) {  // largest x with w(x) > 0
    ln = 31 - __clz(bl);
    rr = __shfl_sync(0xffffffffu, rl, ln);
  } else {         // smallest unchosen site
    ln = __ffs(bf) - 1;
    rr = __shfl_sync(0xffffffffu, rf, ln);
  }
  return (ln - seg * G) * R + rr;
}

// Gauss-Jordan update of one owner's W with the B new rows X_new = pos[k0 .. k0+B) (nb == B
// whenever later columns remain), mapped over (column, row) pairs so that all G lanes work:
//   (1) z_j = V[X_new, j] - V[X_new, 0:k0] W[0:k0, j]           (one lane per (j, t) entry)
//   (2) z_j <- S^{-1} z_j with S = L U from the in-block draws   (one lane per column j)
//   (3) W[0:k0, j] -= W[0:k0, k0:k0+B] z_j,  W[k0+t, j] = z_j[t]  (one lane per (i, j) entry)
// VnT[i][t] = V[x_{k0+t}, m_i] (perm[i] = m_i * stride, the U^T column offset); rows j >= k0+B of
// VnT are overwritten by z_j.
template <int R, int B, int G>
__device__ __forceinline__ void seg_gj_flat(const double* __restrict__ Uts, int stride, const int* perm,
                                            const int* pos, const double* Row, const double* Pinv,
                                            double* Wf, double* VnT, int ldw, int k0, int Np, int sl) {
  using Sw = Swz<double, R>;
  static_assert(G % B == 0, "lane -> t mapping needs B | G");
  static_assert(B % 4 == 0, "step (1) takes four rows per iteration; k0 is a multiple of B");
  const int j0 = k0 + B, nc = Np - j0;
  __syncwarp();
  {
    const int t = sl % B;  // fixed per lane because B | G
    const int xp = Sw::phys(pos[k0 + t]);
    for (int idx = sl; idx < Np * B; idx += G) VnT[idx] = Uts[perm[idx / B] + xp];
  }
  __syncwarp();
  for (int idx = sl; idx < nc * B; idx += G) {
    const int t = idx % B, j = j0 + idx / B;
    // k0 is a multiple of B (>= 4 when nonzero): four independent partial sums
    double a0 = VnT[j * B + t], a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll 2
    for (int ii = 0; ii < k0; ii += 4) {
      a0 = fma(-VnT[ii * B + t], Wf[ii * ldw + j], a0);
      a1 = fma(-VnT[(ii + 1) * B + t], Wf[(ii + 1) * ldw + j], a1);
      a2 = fma(-VnT[(ii + 2) * B + t], Wf[(ii + 2) * ldw + j], a2);
      a3 = fma(-VnT[(ii + 3) * B + t], Wf[(ii + 3) * ldw + j], a3);
    }
    VnT[j * B + t] = (a0 + a1) + (a2 + a3);
  }
  __syncwarp();
  for (int jj = sl; jj < nc; jj += G) {
    const int j = j0 + jj;
    double z[B];
#pragma unroll
    for (int t = 0; t < B; t += 2) {
      const double2 v = *reinterpret_cast<const double2*>(VnT + j * B + t);
      z[t] = v.x;
      z[t + 1] = v.y;
    }
#pragma unroll
    for (int t = 1; t < B; ++t)
#pragma unroll
      for (int t2 = 0; t2 < t; ++t2) z[t] = fma(-(Row[t * B + t2] * Pinv[t2]), z[t2], z[t]);
#pragma unroll
    for (int t = B - 1; t >= 0; --t) {
#pragma unroll
      for (int t2 = t + 1; t2 < B; ++t2) z[t] = fma(-Row[t * B + t2], z[t2], z[t]);
      z[t] *= Pinv[t];
    }
#pragma unroll
    for (int t = 0; t < B; t += 2) *reinterpret_cast<double2*>(VnT + j * B + t) = make_double2(z[t], z[t + 1]);
#pragma unroll
    for (int t = 0; t < B; ++t) Wf[(k0 + t) * ldw + j] = z[t];
  }
  __syncwarp();
  if (k0 > 0) {
    const float rnc = 1.0f / (float)nc;
    const int n = k0 * nc;
#pragma unroll 2
    for (int idx = sl; idx < n; idx += G) {
      int ii = __float2int_rz(((float)idx + 0.5f) * rnc);  // idx / nc (idx < 2^12: exact)
      const int j = j0 + idx - ii * nc;
      double a = Wf[ii * ldw + j], b = 0.0;
#pragma unroll
      for (int t = 0; t < B; t += 2) {
        const double2 wb = *reinterpret_cast<const double2*>(Wf + ii * ldw + k0 + t);
        const double2 zz = *reinterpret_cast<const double2*>(VnT + j * B + t);
        a = fma(-wb.x, zz.x, a);
        b = fma(-wb.y, zz.y, b);
      }
      Wf[ii * ldw + j] = a + b;
    }
  }
  __syncwarp();
}

// OPT bits (development variants, FFS_WARP_VARIANT): 1 = draw keeps its partial sums,
// 2 = pivot row through shared memory (owner lane stores it, no select tree / shuffles),
// 4 = Gauss-Jordan update mapped over (column, row) pairs instead of one lane per column,
// 32 = pivot row by select tree + shuffles (critical columns first), 128 = no vote when G = 32.
template <int R, int B, int G, bool TIMING, int OPT = 0>
__device__ __forceinline__ void ffs_seg_body(const WarpParams& p) {
  extern __shared__ __align__(16) unsigned char smem[];
  using Sw = Swz<double, R>;
  constexpr int SEGS = 32 / G;
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int seg = lane / G, sl = lane % G;
  const int L = p.L, N = p.N, Np = p.Np;
  const int stride = p.ut_stride;

  // ---- U^T into shared memory (swizzled 16-byte chunks; rows >= L zero)
  double* Uts = reinterpret_cast<double*>(smem);
  for (int idx = threadIdx.x; idx < N * p.Lp; idx += blockDim.x) {
    const int x = idx / N, c = idx % N;
    Uts[(size_t)c * stride + Sw::phys(x)] = (x < L) ? p.U[(size_t)x * N + c] : 0.0;
  }
  __syncthreads();

  const WarpLayout lay(Np, B, true);
  const int ldw = lay.ldw;
  unsigned char* ob = smem + p.ushared + (size_t)(wid * SEGS + seg) * p.owner_bytes;
  int* perm = reinterpret_cast<int*>(ob + lay.perm);
  int* pos = reinterpret_cast<int*>(ob + lay.pos);
  double* usel = reinterpret_cast<double*>(ob + lay.usel);
  double* Row = reinterpret_cast<double*>(ob + lay.row);
  double* Pinv = reinterpret_cast<double*>(ob + lay.pinv);
  double* Wf = reinterpret_cast<double*>(ob + lay.wf);
  double* VnT = reinterpret_cast<double*>(ob + lay.vnt);
  const int sw = Sw::sw(sl);
  const double* Ucol0 = Uts + sl * R;
  int qoff[R / 2];  // swizzled 16-byte chunk offsets of this lane's rows within a column
#pragma unroll
  for (int q = 0; q < R / 2; ++q) qoff[q] = (q ^ sw) << 1;
  for (int idx = sl; idx < Np * ldw; idx += G) Wf[idx] = 0.0;  // padding columns stay 0
  for (int idx = sl; idx < B * B; idx += G) Row[idx] = 0.0;
  __syncwarp();

  const int64_t ngroups = (p.M + SEGS - 1) / SEGS;
  long long tacc[TIMING ? 8 : 1] = {0};  // development timing
  for (int64_t g = (int64_t)blockIdx.x * nwarps + wid; g < ngroups; g += (int64_t)gridDim.x * nwarps) {
    const int64_t id = g * SEGS + seg;
    const int64_t i = id < p.M ? id : p.M - 1;  // a short last group recomputes a sample
    for (int j = sl; j < Np; j += G) {
      perm[j] = p.perm[i * Np + j] * stride;  // U^T column offset of m_j
      usel[j] = p.uniforms[i * 2 * (int64_t)Np + Np + j];
    }
    __syncwarp();
    uint32_t chosen = 0;
    int flag = 0;
    constexpr bool tm = TIMING;  // development: per-phase clock64 accounting (separate instance)
    long long tA = 0;
    if constexpr (tm) tA = clock64();

    for (int k0 = 0; k0 < Np; k0 += B) {
      const int nb = min(B, Np - k0);
      // ---- a3 panel: P = V[:, k0:k0+B] - V[:, 0:k0] Wb  (Wb = Wf[0:k0][k0:k0+B], smem)
      double P[R][B];
#pragma unroll
      for (int c = 0; c < B; ++c) {
        const double* cb = Ucol0 + perm[min(k0 + c, Np - 1)];
#pragma unroll
        for (int q = 0; q < R / 2; ++q) {
          const double2 d = *reinterpret_cast<const double2*>(cb + qoff[q]);
          P[2 * q][c] = d.x;
          P[2 * q + 1][c] = d.y;
        }
      }
      if (nb < B) {  // ragged last block: columns past N' are zero
#pragma unroll
        for (int c = 1; c < B; ++c)
          if (c >= nb)
#pragma unroll
            for (int r = 0; r < R; ++r) P[r][c] = 0.0;
      }
      if constexpr ((OPT & 16) != 0) {
        // software-pipelined contraction: operands of row ii+1 (and the permutation entry of
        // ii+2) are loaded before the 2 R B FMAs of row ii are issued
        const int kend = (p.dbg & 1) ? 0 : k0;
        if (kend > 0) {
          double2 ua[R / 2], wa[B / 2];
          int pn = perm[min(1, kend - 1)];
          {
            const double* cb = Ucol0 + perm[0];
#pragma unroll
            for (int q = 0; q < R / 2; ++q) ua[q] = *reinterpret_cast<const double2*>(cb + qoff[q]);
#pragma unroll
            for (int c = 0; c < B; c += 2) wa[c / 2] = *reinterpret_cast<const double2*>(Wf + k0 + c);
          }
          for (int ii = 0; ii < kend; ++ii) {
            const int nx = min(ii + 1, kend - 1);
            const double* cb = Ucol0 + pn;
            pn = perm[min(ii + 2, kend - 1)];
            double2 ub[R / 2], wn[B / 2];
#pragma unroll
            for (int q = 0; q < R / 2; ++q) ub[q] = *reinterpret_cast<const double2*>(cb + qoff[q]);
#pragma unroll
            for (int c = 0; c < B; c += 2) wn[c / 2] = *reinterpret_cast<const double2*>(Wf + nx * ldw + k0 + c);
#pragma unroll
            for (int q = 0; q < R / 2; ++q) {
#pragma unroll
              for (int c = 0; c < B; c += 2) {
                P[2 * q][c] = fma(-ua[q].x, wa[c / 2].x, P[2 * q][c]);
                P[2 * q][c + 1] = fma(-ua[q].x, wa[c / 2].y, P[2 * q][c + 1]);
                P[2 * q + 1][c] = fma(-ua[q].y, wa[c / 2].x, P[2 * q + 1][c]);
                P[2 * q + 1][c + 1] = fma(-ua[q].y, wa[c / 2].y, P[2 * q + 1][c + 1]);
              }
            }
#pragma unroll
            for (int q = 0; q < R / 2; ++q) ua[q] = ub[q];
#pragma unroll
            for (int c = 0; c < B / 2; ++c) wa[c] = wn[c];
          }
        }
      } else {
        const int kend = (p.dbg & 1) ? 0 : k0;
        const double* wrow = Wf + k0;
#pragma unroll 2
        for (int ii = 0; ii < kend; ++ii, wrow += ldw) {
          const double* cb = Ucol0 + perm[ii];
          double wb[B];
#pragma unroll
          for (int c = 0; c < B; c += 2) {
            const double2 d = *reinterpret_cast<const double2*>(wrow + c);
            wb[c] = d.x;
            wb[c + 1] = d.y;
          }
#pragma unroll
          for (int q = 0; q < R / 2; ++q) {
            const double2 d = *reinterpret_cast<const double2*>(cb + qoff[q]);
#pragma unroll
            for (int c = 0; c < B; ++c) {
              P[2 * q][c] = fma(-d.x, wb[c], P[2 * q][c]);
              P[2 * q + 1][c] = fma(-d.y, wb[c], P[2 * q + 1][c]);
            }
          }
        }
      }
      // rows drawn in earlier blocks: exactly zero (the contraction leaves O(eps) residues)
      // rows drawn earlier get weight exactly 0: mask the column of the next draw (only that
      // column is ever squared; the contraction leaves O(eps) residues in drawn rows)
      if constexpr ((OPT & 512) == 0) {
#pragma unroll
        for (int r = 0; r < R; ++r) P[r][0] = ((chosen >> r) & 1u) ? 0.0 : P[r][0];
      }
      if constexpr (tm) {
        const long long t = clock64();
        tacc[0] += (t - tA);
        tA = t;
      }

      // ---- a4/a5: nb sequential draws on the panel, one-column lookahead
      Draw dr;
      {
        double col0[R];
#pragma unroll
        for (int r = 0; r < R; ++r) col0[r] = P[r][0];
        if (p.dbg & 2) { dr.ball = 1u; dr.rsel = (k0 / B) % R; dr.T = 1.0; }
        else dr = seg_draw<R, G, (OPT & 1) != 0>(col0, usel[k0], seg);
      }
      static_for<0, B>([&](auto rrc) {
        constexpr int rr = decltype(rrc)::value;
        if (rr < nb) {
          const int k = k0 + rr;
          long long ts0 = 0;
          if constexpr (tm) ts0 = clock64();
          int own, orow = 0;  // owner lane within the segment, row within the owner
          // G == 32: one segment per warp, dr.ball is warp-uniform (no vote needed)
          bool common;
          if constexpr (G == 32 && (OPT & 160) != 0) common = dr.ball != 0u;
          else common = __all_sync(0xffffffffu, dr.ball != 0u);
          if constexpr ((OPT & 512) != 0) {
            // rows drawn earlier are not masked (they hold O(eps) residues of weight ~eps^2 T):
            // a crossing on such a row, or no crossing at all, takes the exact masked redraw
            static_assert(G == 32, "OPT 512 is written for one segment per warp");
            own = __ffs(dr.ball) - 1;
            common = common && !__any_sync(0xffffffffu, (lane == own) && ((chosen >> dr.rsel) & 1u));
            if (!common) {
              double colr[R];
#pragma unroll
              for (int r = 0; r < R; ++r) colr[r] = ((chosen >> r) & 1u) ? 0.0 : P[r][rr];
              dr = seg_draw<R, G, (OPT & 1) != 0>(colr, usel[k], seg);
              if (dr.ball != 0u) {
                own = __ffs(dr.ball) - 1;
                orow = __shfl_sync(0xffffffffu, dr.rsel, own);
              } else {
                const int xf = seg_fallback<R, G>(colr, dr.T, chosen, L, sl, seg);
                own = xf / R;
                orow = xf % R;
              }
            }
          } else if (common) {
            own = __ffs(dr.ball) - 1;
            if constexpr (!(OPT & 34)) orow = __shfl_sync(0xffffffffu, dr.rsel, seg * G + own);
          } else {
            // rare: some segment has u*T at/after its last partial sum, or T not finite/positive
            int o = 0, rw = 0;
            if (dr.ball != 0u) {
              o = __ffs(dr.ball) - 1;
            }
            rw = __shfl_sync(0xffffffffu, dr.rsel, seg * G + o);
            double colr[R];
#pragma unroll
            for (int r = 0; r < R; ++r) colr[r] = P[r][rr];
            const int xf = seg_fallback<R, G>(colr, dr.T, chosen, L, sl, seg);
            own = dr.ball != 0u ? o : xf / R;
            orow = dr.ball != 0u ? rw : xf % R;
          }
          if constexpr (tm) {
            const long long t = clock64() + (long long)orow * 0;
            tacc[3] += (t - ts0);
            ts0 = t;
          }
          if (!((dr.T > 0.0) && (dr.T <= 1.7976931348623157e308))) flag |= 1;
          if (p.trace != nullptr && id < p.S) {
            const double inv = dr.T > 0.0 ? 1.0 / dr.T : 0.0;
            double* tr = p.trace + (id * Np + k) * (int64_t)L;
#pragma unroll
            for (int r = 0; r < R; ++r)
              if (sl * R + r < L) tr[sl * R + r] = P[r][rr] * P[r][rr] * inv;
          }
          // pivot row: every lane selects row `rs` of its own R x B block with a branch-free
          // select tree (rs = its crossing row, or orow on the rare fallback path); the owner
          // lane's selection is then broadcast to its segment with shuffles (no smem, no branch)
          const double Tk = dr.T;
          const int rs = (OPT & 512) ? (common ? dr.rsel : orow) : (dr.ball != 0u ? dr.rsel : orow);
          double pv;  // pivot P[x_k][rr]
          double prow[B];
          if constexpr ((OPT & 512) != 0) {
            // only the owner lane branches into the store of its row rs (8-way switch, 64-bit
            // stores: no register shuffling into 128-bit groups, no predicated stores elsewhere)
            if (sl == own) {
              double* dst = Row + rr * B;
              switch (rs) {
#define FFS_ROWST(RR) case RR: _Pragma("unroll") for (int c = 0; c < B; ++c) if (RR < R) dst[c] = P[RR < R ? RR : 0][c]; break;
                FFS_ROWST(0) FFS_ROWST(1) FFS_ROWST(2) FFS_ROWST(3) FFS_ROWST(4) FFS_ROWST(5) FFS_ROWST(6) FFS_ROWST(7)
#undef FFS_ROWST
                default: break;
              }
              pos[k] = own * R + rs;
            }
            chosen |= (sl == own) ? (1u << rs) : 0u;
            __syncwarp();
            pv = Row[rr * B + rr];
          } else if constexpr ((OPT & 32) != 0) {
            // columns rr and rr+1 first: they feed the reciprocal and the next column's update
            // (the critical path); the others only feed the in-block updates and Row
            auto extract = [&](int c) {
              double t[R];
#pragma unroll
              for (int r = 0; r < R; ++r) t[r] = P[r][c];
#pragma unroll
              for (int w = 1; w < R; w <<= 1)
#pragma unroll
                for (int i = 0; i < R; i += 2 * w) t[i] = (rs & w) ? t[i + w] : t[i];
              return __shfl_sync(0xffffffffu, t[0], seg * G + own);
            };
            prow[rr] = extract(rr);
            if constexpr (rr + 1 < B) prow[rr + 1] = extract(rr + 1);
#pragma unroll
            for (int c = 0; c < B; ++c)
              if (c != rr && c != rr + 1) prow[c] = extract(c);
            chosen |= (sl == own) ? (1u << rs) : 0u;
            if (sl == own) pos[k] = own * R + rs;
            if (sl == 0) {
#pragma unroll
              for (int c = 0; c < B; c += 2)
                *reinterpret_cast<double2*>(Row + rr * B + c) = make_double2(prow[c], prow[c + 1]);
            }
            pv = prow[rr];
          } else if constexpr ((OPT & 2) != 0) {
            // the owner lane stores row rs of its block (the row it selected itself) into Row
            const bool mine = (sl == own);
#pragma unroll
            for (int r = 0; r < R; ++r)
              if (mine && r == rs) {
#pragma unroll
                for (int c = 0; c < B; c += 2)
                  *reinterpret_cast<double2*>(Row + rr * B + c) = make_double2(P[r][c], P[r][c + 1]);
              }
            if (mine) pos[k] = own * R + rs;
            chosen |= mine ? (1u << rs) : 0u;
            __syncwarp();
            pv = Row[rr * B + rr];
          } else {
#pragma unroll
            for (int c = 0; c < B; ++c) {
              double t[R];
#pragma unroll
              for (int r = 0; r < R; ++r) t[r] = P[r][c];
#pragma unroll
              for (int w = 1; w < R; w <<= 1)
#pragma unroll
                for (int i = 0; i < R; i += 2 * w) t[i] = (rs & w) ? t[i + w] : t[i];
              prow[c] = __shfl_sync(0xffffffffu, t[0], seg * G + own);
            }
            chosen |= (sl == own) ? (1u << orow) : 0u;
            if (sl == 0) {
              pos[k] = own * R + orow;
#pragma unroll
              for (int c = 0; c < B; c += 2)
                *reinterpret_cast<double2*>(Row + rr * B + c) = make_double2(prow[c], prow[c + 1]);
            }
            pv = prow[rr];
          }
          if (pv * pv < 1e-12 * Tk) flag |= 2;
          if constexpr (tm) {
            const long long t = clock64() + (long long)(pv * 0.0);
            tacc[4] += (t - ts0);
            ts0 = t;
          }
          const double ip = fast_rcp(pv);
          if constexpr (tm) {
            const long long t = clock64() + (long long)(ip * 0.0);
            tacc[5] += (t - ts0);
            ts0 = t;
          }
          if (sl == 0) Pinv[rr] = ip;
          if constexpr (rr + 1 < B) {
            double sp[B];  // pivot row scaled by 1/pivot
            if constexpr ((OPT & 32) != 0) {
#pragma unroll
              for (int c = 0; c < B; ++c) sp[c] = prow[c] * ip;
            } else {
#pragma unroll
              for (int c = 0; c < B; c += 2) {
                const double2 d = *reinterpret_cast<const double2*>(Row + rr * B + c);
                sp[c] = d.x * ip;
                sp[c + 1] = d.y * ip;
              }
            }
            // column rr+1 first, then the next draw, then the remaining columns
#pragma unroll
            for (int r = 0; r < R; ++r) {
              if constexpr ((OPT & 512) != 0) P[r][rr + 1] = fma(-P[r][rr], sp[rr + 1], P[r][rr + 1]);
              else P[r][rr + 1] = ((chosen >> r) & 1u) ? 0.0 : fma(-P[r][rr], sp[rr + 1], P[r][rr + 1]);
            }
            if (rr + 1 < nb) {
              double cn[R];
#pragma unroll
              for (int r = 0; r < R; ++r) cn[r] = P[r][rr + 1];
              if (p.dbg & 2) { dr.ball = 1u << ((k + 1) % G); dr.rsel = (k + 1) / G % R; dr.T = 1.0 + cn[0] * 1e-300; }
              else dr = seg_draw<R, G, (OPT & 1) != 0>(cn, usel[k + 1], seg);
              if constexpr (tm) {
                const long long t = clock64() + (long long)(dr.T * 0.0) + dr.rsel * 0;
                tacc[6] += (t - ts0);
                ts0 = t;
              }
            }
#pragma unroll
            for (int c = rr + 2; c < B; ++c)
#pragma unroll
              for (int r = 0; r < R; ++r) P[r][c] = fma(-P[r][rr], sp[c], P[r][c]);
          }
        }
      });

      if constexpr (tm) {
        const long long t = clock64();
        tacc[1] += (t - tA);
        tA = t;
      }
      // ---- Gauss-Jordan update of W with the nb new rows (only if later columns remain)
      if constexpr ((OPT & 4) != 0) {
        if (k0 + nb < Np && !(p.dbg & 4)) seg_gj_flat<R, B, G>(Uts, stride, perm, pos, Row, Pinv, Wf, VnT, ldw, k0, Np, sl);
      } else if (k0 + nb < Np && !(p.dbg & 4)) {
        __syncwarp();
        for (int idx = sl; idx < Np * B; idx += G) {
          const int ii = idx / B, tt = idx % B;
          VnT[idx] = (tt < nb) ? Uts[perm[ii] + Sw::phys(pos[k0 + tt])] : 0.0;
        }
        __syncwarp();
        for (int j = k0 + nb + sl; j < Np; j += G) {
          double z[B];
#pragma unroll
          for (int tt = 0; tt < B; ++tt) z[tt] = VnT[j * B + tt];
#pragma unroll 2
          for (int ii = 0; ii < k0; ++ii) {
            const double wij = Wf[ii * ldw + j];
#pragma unroll
            for (int tt = 0; tt < B; tt += 2) {
              const double2 v = *reinterpret_cast<const double2*>(VnT + ii * B + tt);
              z[tt] = fma(-v.x, wij, z[tt]);
              z[tt + 1] = fma(-v.y, wij, z[tt + 1]);
            }
          }
          double ipv[B];
#pragma unroll
          for (int t2 = 0; t2 < B; ++t2) ipv[t2] = (t2 < nb) ? Pinv[t2] : 0.0;
#pragma unroll
          for (int tt = 1; tt < B; ++tt)
#pragma unroll
            for (int t2 = 0; t2 < tt; ++t2) z[tt] = fma(-(Row[tt * B + t2] * ipv[t2]), z[t2], z[tt]);
#pragma unroll
          for (int tt = B - 1; tt >= 0; --tt) {
#pragma unroll
            for (int t2 = tt + 1; t2 < B; ++t2) z[tt] = fma(-Row[tt * B + t2], z[t2], z[tt]);
            z[tt] *= ipv[tt];
          }
#pragma unroll 2
          for (int ii = 0; ii < k0; ++ii) {
            double a = Wf[ii * ldw + j];
#pragma unroll
            for (int tt = 0; tt < B; tt += 2) {
              const double2 wbv = *reinterpret_cast<const double2*>(Wf + ii * ldw + k0 + tt);
              a = fma(-wbv.x, z[tt], a);
              a = fma(-wbv.y, z[tt + 1], a);
            }
            Wf[ii * ldw + j] = a;
          }
#pragma unroll
          for (int tt = 0; tt < B; ++tt)
            if (tt < nb) Wf[(k0 + tt) * ldw + j] = z[tt];
        }
        __syncwarp();
      }
      if constexpr (tm) {
        const long long t = clock64();
        tacc[2] += (t - tA);
        tA = t;
      }
    }
    // ---- a6: positions and flags
    unsigned fl = __reduce_or_sync(0xffffffffu, (unsigned)flag << (seg * 2));
    if (id < p.M) {
      for (int j = sl; j < Np; j += G) p.positions[id * Np + j] = pos[j];
      if (sl == 0 && p.flags != nullptr) p.flags[id] = (fl >> (seg * 2)) & 3u;
    }
    __syncwarp();
  }
  if constexpr (TIMING) {
    if (p.timing != nullptr && lane == 0)
      for (int q = 0; q < 8; ++q) atomicAdd(p.timing + q, (unsigned long long)tacc[q]);
  }
}

template <int R, int B, int G, int MAXT, bool TIMING = false, int OPT = 0>
__global__ void __launch_bounds__(MAXT, 1) ffs_seg_kernel(const WarpParams p) {
  ffs_seg_body<R, B, G, TIMING, OPT>(p);
}

}  // namespace ffsk
