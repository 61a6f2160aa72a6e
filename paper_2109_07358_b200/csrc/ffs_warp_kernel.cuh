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
  size_t perm, pos, usel, row, pinv, wf, vnt, total;
  int ldw;  // row stride of W: N'+2 (B | N') or N'+B, rounded to even; columns [N', ldw) stay zero
  __host__ __device__ WarpLayout(int Np, int B) {
    // (Np + 2 when B | N': rows of W start 16 bytes apart in bank space, so the flat
    // Gauss-Jordan mapping's (row, column) accesses do not collide)
    ldw = (Np % B == 0) ? ((Np + 3) & ~1) : ((Np + B + 1) & ~1);
    size_t o = 0;
    perm = o; o = align16(o + sizeof(int) * Np);
    pos = o;  o = align16(o + sizeof(int) * Np);
    usel = o; o = align16(o + sizeof(double) * Np);
    row = o;  o = align16(o + sizeof(double) * B * B);
    pinv = o; o = align16(o + sizeof(double) * B);
    wf = o;   o = align16(o + sizeof(double) * (size_t)Np * ldw);
    vnt = o;  o = align16(o + sizeof(double) * (size_t)Np * B);
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
  int64_t S0, S;           // debug trace of samples S0 .. S0+S-1
  double* trace;          // [S][Np][L] or null
};

// Result of the branch-free part of a draw.
struct Draw {
  unsigned ball;  // lanes whose inclusive prefix exceeds u*T (the crossing lane is the first)
  int rsel;       // in the crossing lane: the first row with C(x) > u*T
  double T;       // total weight
};

// U [L][N] -> per-sample permutation prefix [M][Np] (a1 rule, reading Q6); one thread per sample.
static __global__ void ffs_permute_kernel(const double* __restrict__ uniforms, int64_t ustride,
                                          int32_t* __restrict__ perm, int64_t M, int N, int Np) {
  extern __shared__ int pscratch[];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // per-thread working permutation, interleaved across the block ([N][blockDim]): the threads of
  // a warp touch 32 consecutive words (no bank conflicts)
  int* m = pscratch + threadIdx.x;
  const int bs = blockDim.x;
  if (i >= M) return;
  for (int j = 0; j < N; ++j) m[j * bs] = j;
  const double* u = uniforms + i * ustride;
  for (int j = 0; j < Np; ++j) {
    const int n = N - j;
    int r = (int)floor(u[j] * (double)n);
    r = (r > n - 1 ? n - 1 : r) + j;
    FFS_CHECK(r >= j && r < N);
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

// Branch-free part of a draw for one segment: the crossing lanes of this lane's segment (bit i =
// segment lane i), the crossing row in this lane, and T. The lane's partial sums are kept in
// registers, so the row search after the ballot is R-1 independent compares. Every prefix value
// compared against the threshold is the previous lane's inclusive value plus this lane's own
// partial sums, so the crossing lane and row are consistent (reading Q5).
template <int R, int G>
__device__ __forceinline__ Draw seg_draw(const double (&col)[R], double u, int seg) {
  static_assert(R <= 8, "row search keeps R partial sums in registers");
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
  // crossing threshold relative to this lane's exclusive prefix, clamped at 0 so that a lane
  // whose rounded prefix already passed u*T still lands on its first positive weight
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

// One sample per G-lane segment (profiles/r01_ncu_summary.md for the measured
// alternatives): the draw keeps its partial sums, the owner lane stores the pivot row to shared
// memory (no select tree), the Gauss-Jordan update is mapped over (column, row) pairs, and a
// whole-warp segment (G = 32) needs no warp vote before the common path.
template <int R, int B, int G>
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

  const WarpLayout lay(Np, B);
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
  for (int64_t g = (int64_t)blockIdx.x * nwarps + wid; g < ngroups; g += (int64_t)gridDim.x * nwarps) {
    const int64_t id = g * SEGS + seg;
    const int64_t i = id < p.M ? id : p.M - 1;  // a short last group recomputes a sample
    for (int j = sl; j < Np; j += G) {
      FFS_CHECK(p.perm[i * Np + j] >= 0 && p.perm[i * Np + j] < N);
      perm[j] = p.perm[i * Np + j] * stride;  // U^T column offset of m_j
      usel[j] = p.uniforms[i * 2 * (int64_t)Np + Np + j];
    }
    __syncwarp();
    uint32_t chosen = 0;
    int flag = 0;

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
      {
        const double* wrow = Wf + k0;
#pragma unroll 2
        for (int ii = 0; ii < k0; ++ii, wrow += ldw) {
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
      // rows drawn earlier get weight exactly 0: mask the column of the next draw (only that
      // column is ever squared; the contraction leaves O(eps) residues in drawn rows)
#pragma unroll
      for (int r = 0; r < R; ++r) P[r][0] = ((chosen >> r) & 1u) ? 0.0 : P[r][0];

      // ---- a4/a5: nb sequential draws on the panel, one-column lookahead
      Draw dr;
      {
        double col0[R];
#pragma unroll
        for (int r = 0; r < R; ++r) col0[r] = P[r][0];
        dr = seg_draw<R, G>(col0, usel[k0], seg);
      }
      static_for<0, B>([&](auto rrc) {
        constexpr int rr = decltype(rrc)::value;
        if (rr < nb) {
          const int k = k0 + rr;
          int own, orow = 0;  // owner lane within the segment, row within the owner (rare path)
          // G == 32: one segment per warp, dr.ball is warp-uniform (no vote needed)
          bool common;
          if constexpr (G == 32) common = dr.ball != 0u;
          else common = __all_sync(0xffffffffu, dr.ball != 0u);
          if (common) {
            own = __ffs(dr.ball) - 1;
          } else {
            // rare: some segment has u*T at/after its last partial sum, or T not finite/positive
            int o = 0, rw = 0;
            if (dr.ball != 0u) o = __ffs(dr.ball) - 1;
            rw = __shfl_sync(0xffffffffu, dr.rsel, seg * G + o);
            double colr[R];
#pragma unroll
            for (int r = 0; r < R; ++r) colr[r] = P[r][rr];
            const int xf = seg_fallback<R, G>(colr, dr.T, chosen, L, sl, seg);
            own = dr.ball != 0u ? o : xf / R;
            orow = dr.ball != 0u ? rw : xf % R;
          }
          if (!((dr.T > 0.0) && (dr.T <= 1.7976931348623157e308))) flag |= 1;
          if (p.trace != nullptr && (uint64_t)(id - p.S0) < (uint64_t)p.S) {
            const double inv = dr.T > 0.0 ? 1.0 / dr.T : 0.0;
            double* tr = p.trace + ((id - p.S0) * Np + k) * (int64_t)L;
#pragma unroll
            for (int r = 0; r < R; ++r)
              if (sl * R + r < L) tr[sl * R + r] = P[r][rr] * P[r][rr] * inv;
          }
          // pivot row: the owner lane stores row rs of its block (the row it selected itself)
          const double Tk = dr.T;
          const int rs = dr.ball != 0u ? dr.rsel : orow;
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
          const double pv = Row[rr * B + rr];  // pivot P[x_k][rr]
          if (pv * pv < 1e-12 * Tk) flag |= 2;
          const double ip = fast_rcp(pv);
          if (sl == 0) Pinv[rr] = ip;
          if constexpr (rr + 1 < B) {
            double sp[B];  // pivot row scaled by 1/pivot
#pragma unroll
            for (int c = 0; c < B; c += 2) {
              const double2 d = *reinterpret_cast<const double2*>(Row + rr * B + c);
              sp[c] = d.x * ip;
              sp[c + 1] = d.y * ip;
            }
            // column rr+1 first, then the next draw, then the remaining columns
#pragma unroll
            for (int r = 0; r < R; ++r)
              P[r][rr + 1] = ((chosen >> r) & 1u) ? 0.0 : fma(-P[r][rr], sp[rr + 1], P[r][rr + 1]);
            if (rr + 1 < nb) {
              double cn[R];
#pragma unroll
              for (int r = 0; r < R; ++r) cn[r] = P[r][rr + 1];
              dr = seg_draw<R, G>(cn, usel[k + 1], seg);
            }
#pragma unroll
            for (int c = rr + 2; c < B; ++c)
#pragma unroll
              for (int r = 0; r < R; ++r) P[r][c] = fma(-P[r][rr], sp[c], P[r][c]);
          }
        }
      });

      // ---- Gauss-Jordan update of W with the nb new rows (only if later columns remain)
      if (k0 + nb < Np) seg_gj_flat<R, B, G>(Uts, stride, perm, pos, Row, Pinv, Wf, VnT, ldw, k0, Np, sl);
    }
    // ---- a6: positions and flags
    unsigned fl = __reduce_or_sync(0xffffffffu, (unsigned)flag << (seg * 2));
    if (id < p.M) {
      for (int j = sl; j < Np; j += G) {
        FFS_CHECK(pos[j] >= 0 && pos[j] < L);
        p.positions[id * Np + j] = pos[j];
      }
      if (sl == 0 && p.flags != nullptr) p.flags[id] = (fl >> (seg * 2)) & 3u;
    }
    __syncwarp();
  }
}

template <int R, int B, int G, int MAXT>
__global__ void __launch_bounds__(MAXT, 1) ffs_seg_kernel(const WarpParams p) {
  ffs_seg_body<R, B, G>(p);
}

}  // namespace ffsk
