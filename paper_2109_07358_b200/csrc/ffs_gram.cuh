// Gram-matrix draws for the block-step paths (a4/a5 of one block step, every batch sample).
//
// One block step draws B = 8 sites x_{k0..k0+7} of a sample from its L x B panel P (the Schur
// complement columns k0..k0+7 after the first k0 draws; ffs_dense.cuh). Draw r of the block has
// the weights (Eq. 3)
//   w_r(x) = |s_r(x)|^2,   s_r(x) = P[x,r] - P[x,0:r] c_r = sum_{q<=r} P[x,q] d_r[q],
//   c_r = A^{-1} P[X,r],  A = P[X_{0..r-1}, 0:r],  d_r = (-c_r; 1)
// (the right-looking rank-1 updates of the other kernels, written as one combination of the
// ORIGINAL panel columns). Sums of w_r over any set of rows are therefore quadratic forms of the
// Gram matrix of the panel restricted to that set:
//   sum_{x in tile} w_r(x) = d_r^H G_tile d_r,   G_tile[q][q'] = sum_{x in tile} conj(P[x,q]) P[x,q'].
// ffs_gram_kernel forms G for 32 row tiles per sample in one pass over the panel (HBM-bound);
// ffs_gram_draw_kernel then runs the 8 draws of a sample in ONE WARP: lane t evaluates tile t's
// total (a dot product of <= 36 real / 64 complex terms), a warp scan finds the tile the threshold
// u T falls in, and only that tile's rows (L/32) are read and scanned to find x_k. No panel lives
// in registers, no cluster or CTA barrier is involved, and ~16 samples per SM are in flight
// instead of one per 8 SMs (profiles/r02_ncu_summary.md: the cluster step kernel spent ~8 K cycles
// per draw, half of it in cluster barriers).
//
// Rounding: the quadratic form cancels when |d| is large (a small in-block pivot). Its absolute
// error is bounded by ~eps (sum_q |d_q| sqrt(G[q][q]))^2 =: eps * bound; when T < bound / kappa_max the
// warp recomputes the 32 tile totals directly from the panel rows (exact to summation rounding)
// before it selects -- so the CDF the draw uses is within ~36 eps kappa_max T of the exact one,
// inside the 1e-9 tie window of reading Q10. Rows already drawn weigh exactly 0 (bitmap /
// in-block list), as in every other path.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ffs_kernel.cuh"

namespace ffsk {

// Upper-triangle entry layout, column-major by q' so that draw r uses a PREFIX of the entries:
// real: e(q, q') = q'(q'+1)/2 + q (q <= q'); complex: column q' starts at q'^2 with the (real)
// diagonal, then (Re, Im) of G[q][q'] for q < q'.
template <typename T> struct GramIdx;
template <> struct GramIdx<double> {
  static constexpr int NE = 36;
  __host__ __device__ static constexpr int count(int r) { return (r + 1) * (r + 2) / 2; }
};
template <> struct GramIdx<cplx> {
  static constexpr int NE = 64;
  __host__ __device__ static constexpr int count(int r) { return (r + 1) * (r + 1); }
};

struct GramParams {
  const double* Pd;          // [Sb][L][B] panels (scalars of T)
  double* G;                 // [Sb][NE][32] tile Gram entries (lane-minor)
  uint32_t* chosen_g;        // [Sb][Lpt/32] rows drawn so far
  const double* uniforms;    // [M][2Np]
  int32_t* positions;        // [M][Np]
  int32_t* flags;            // [M] or null
  double* rowg;              // [Sb][B*B + B] pivot rows / inverse pivots of this block (out)
  int L, Lpt, Np, Sb, Rt, k0;  // Rt rows per tile (multiple of 32, 32 Rt >= L)
  int64_t base, S0, S;
  double* trace;             // [S][Np][L] or null
  unsigned long long* stats; // [2] draws, direct-sum recomputations (or null)
  double kappa_max;
};

__device__ unsigned long long g_gram_stats[2];

// Sum of v[e] over the 32 lanes for 64 values by recursive halving: at the step with lane mask
// 16, 8, .., 1 a lane keeps the half of its values selected by that lane bit and receives the
// partner's sums of that half (32 + 16 + .. + 2 = 62 shuffles instead of 64 x 5); afterwards lane l
// holds the totals of entries 2 l and 2 l + 1 in v[0], v[1].
__device__ __forceinline__ void warp_reduce_scatter64(double (&v)[64], int lane) {
#pragma unroll
  for (int h = 32; h >= 2; h >>= 1) {
    const bool up = (lane & (h >> 1)) != 0;
#pragma unroll
    for (int j = 0; j < h; ++j) {
      const double send = up ? v[j] : v[j + h];
      const double keep = up ? v[j + h] : v[j];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, h >> 1);
    }
  }
}

// one warp per (sample, tile): lane l takes rows l, l + 32, ... of the tile
template <typename T, int B>
static __global__ void __launch_bounds__(256) ffs_gram_kernel(const GramParams p) {
  constexpr int NE = GramIdx<T>::NE;
  constexpr int kD = Sc<T>::kDoubles;
  constexpr int kV = B * kD / 2;  // 16-byte vectors per row
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t wid = (int64_t)blockIdx.x * 8 + warp;
  if (wid >= (int64_t)p.Sb * 32) return;
  const int sl = (int)(wid >> 5), tau = (int)(wid & 31);
  const int L = p.L;
  const double2* Ps = reinterpret_cast<const double2*>(reinterpret_cast<const T*>(p.Pd) + (size_t)sl * L * B);
  const uint32_t* ch = p.chosen_g + (size_t)sl * (p.Lpt / 32);
  double acc[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) acc[e] = 0.0;
  const int r0 = tau * p.Rt;
  const int r1 = min(L, r0 + p.Rt);
#pragma unroll 2
  for (int xb = r0; xb < r1; xb += 32) {
    const int x = xb + lane;
    const uint32_t cw = ch[xb >> 5];
    const bool act = x < L && !((cw >> lane) & 1u);
    double v[B * kD];
    const double2* pr = Ps + (size_t)(x < L ? x : L - 1) * kV;
#pragma unroll
    for (int j = 0; j < kV; ++j) {
      const double2 d2 = pr[j];
      v[2 * j] = act ? d2.x : 0.0;
      v[2 * j + 1] = act ? d2.y : 0.0;
    }
    if constexpr (kD == 1) {
#pragma unroll
      for (int b = 0; b < B; ++b)
#pragma unroll
        for (int a = 0; a <= b; ++a) acc[b * (b + 1) / 2 + a] = fma(v[a], v[b], acc[b * (b + 1) / 2 + a]);
    } else {
#pragma unroll
      for (int b = 0; b < B; ++b) {
        const double br = v[2 * b], bi = v[2 * b + 1];
        acc[b * b] = fma(br, br, fma(bi, bi, acc[b * b]));
#pragma unroll
        for (int a = 0; a < b; ++a) {
          const double ar = v[2 * a], ai = v[2 * a + 1];
          // conj(P_a) P_b
          acc[b * b + 1 + 2 * a] = fma(ar, br, fma(ai, bi, acc[b * b + 1 + 2 * a]));
          acc[b * b + 2 + 2 * a] = fma(ar, bi, fma(-ai, br, acc[b * b + 2 + 2 * a]));
        }
      }
    }
  }
  double* out = p.G + (size_t)sl * NE * 32 + tau;
  double v64[64];
#pragma unroll
  for (int e = 0; e < 64; ++e) v64[e] = e < NE ? acc[e] : 0.0;
  warp_reduce_scatter64(v64, lane);
  if (2 * lane < NE) out[(size_t)(2 * lane) * 32] = v64[0];
  if (2 * lane + 1 < NE) out[(size_t)(2 * lane + 1) * 32] = v64[1];
}

template <typename T, int B>
struct GramWarpSmem {
  double Gs[GramIdx<T>::NE][32];
  double coef[GramIdx<T>::NE];
  T Row[B][B];
  T Pinv[B];
  T C[B][B];  // C[q][c] = (A^{-1} P[X, c])_q for the rows drawn so far in this block
  T xrow[B];
};

constexpr int kGramWarps = 4;
constexpr int kGramMaxRl = 16;  // rows per lane of a tile: L <= 16384

template <typename T, int B>
static __global__ void __launch_bounds__(32 * kGramWarps) ffs_gram_draw_kernel(const GramParams p) {
  using S = Sc<T>;
  using GI = GramIdx<T>;
  constexpr int NE = GI::NE, kD = S::kDoubles;
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sl = blockIdx.x * kGramWarps + warp;
  if (sl >= p.Sb) return;  // warps are independent (warp-level synchronisation only)
  GramWarpSmem<T, B>& sm = reinterpret_cast<GramWarpSmem<T, B>*>(smem)[warp];
  const int64_t i = p.base + sl;
  const int L = p.L, Np = p.Np, k0 = p.k0, Rt = p.Rt, Rl = Rt >> 5;
  const int nb = min(B, Np - k0);
  const T* Ps = reinterpret_cast<const T*>(p.Pd) + (size_t)sl * L * B;
  uint32_t* ch = p.chosen_g + (size_t)sl * (p.Lpt / 32);
  const double* usel = p.uniforms + i * 2 * (int64_t)Np + Np;
  {
    const double* Gg = p.G + (size_t)sl * NE * 32;
#pragma unroll 8
    for (int e = 0; e < NE; ++e) sm.Gs[e][lane] = Gg[e * 32 + lane];
    for (int idx = lane; idx < B * B; idx += 32) {
      (&sm.Row[0][0])[idx] = S::zero();
      (&sm.C[0][0])[idx] = S::zero();
    }
    if (lane < B) sm.Pinv[lane] = S::zero();
  }
  __syncwarp();
  // sqrt(G[q][q]) of this lane's tile: the rounding scale of the forms (|G[q][q']| <= sg[q] sg[q'], and
  // the accumulated entries carry errors of that size)
  double sg[B];
#pragma unroll
  for (int q = 0; q < B; ++q) sg[q] = sqrt(fmax(sm.Gs[kD == 1 ? q * (q + 1) / 2 + q : q * q][lane], 0.0));
  int xsv[B];
#pragma unroll
  for (int q = 0; q < B; ++q) xsv[q] = -1;
  int flag = 0;
  unsigned ndirect = 0;
  const bool traced = p.trace != nullptr && (uint64_t)(i - p.S0) < (uint64_t)p.S;

  static_for<0, B>([&](auto rc) {
    constexpr int r = decltype(rc)::value;
    if (r < nb) {
      const int k = k0 + r;
      const double u = usel[k];
      // c_r (uniform): dn[q] = C[q][r]
      T dn[r > 0 ? r : 1];
#pragma unroll
      for (int q = 0; q < r; ++q) dn[q] = sm.C[q][r];
      // ---- coefficients of the quadratic form (lane q' fills column q')
      if (lane <= r) {
        const int qp = lane;
        const T dqp = qp == r ? S::one() : S::neg(sm.C[qp][r]);
        for (int q = 0; q <= qp; ++q) {
          const T dq = q == r ? S::one() : S::neg(sm.C[q][r]);
          if constexpr (kD == 1) {
            sm.coef[qp * (qp + 1) / 2 + q] = q == qp ? dq * dq : 2.0 * dq * dqp;
          } else {
            if (q == qp) {
              sm.coef[qp * qp] = S::abs2(dq);
            } else {  // e = conj(d_q) d_q'
              sm.coef[qp * qp + 1 + 2 * q] = 2.0 * fma(dq.re, dqp.re, dq.im * dqp.im);
              sm.coef[qp * qp + 2 + 2 * q] = -2.0 * fma(dq.re, dqp.im, -dq.im * dqp.re);
            }
          }
        }
      }
      __syncwarp();
      // ---- tile totals f (lane = tile) and their rounding scale
      double f = 0.0;
#pragma unroll
      for (int e = 0; e < GI::count(r); ++e) f = fma(sm.coef[e], sm.Gs[e][lane], f);
      if (f < 0.0) f = 0.0;
      // bound of sum |d_q||d_q'||G[q][q']| for this tile: (sum_q |d_q| sqrt(G[q][q]))^2
      double bd = sg[r];
#pragma unroll
      for (int q = 0; q < r; ++q) bd = fma(sqrt(S::abs2(dn[q])), sg[q], bd);
      bd *= bd;

      auto masked = [&](int x) -> bool {
        bool m = ((ch[x >> 5] >> (x & 31)) & 1u) != 0u;
#pragma unroll
        for (int q = 0; q < r; ++q) m = m || x == xsv[q];
        return m;
      };
      // |s_r(x)|^2 from the original panel row (x < L)
      auto weight = [&](int x) -> double {
        constexpr int nv = ((r + 1) * kD + 1) / 2;
        const double2* pr = reinterpret_cast<const double2*>(Ps + (size_t)x * B);
        double2 v2[nv];
#pragma unroll
        for (int j = 0; j < nv; ++j) v2[j] = pr[j];
        auto col = [&](int q) -> T {
          if constexpr (kD == 1) return (q & 1) ? v2[q >> 1].y : v2[q >> 1].x;
          else return cplx{v2[q].x, v2[q].y};
        };
        T s = col(r);
#pragma unroll
        for (int q = 0; q < r; ++q) s = S::fms(col(q), dn[q], s);
        return S::abs2(s);
      };
      auto scan = [&](double v) -> double {
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const double y = __shfl_up_sync(0xffffffffu, v, d);
          if (lane >= d) v += y;
        }
        return v;
      };

      double incl = f, bt = bd;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += y;
        bt += __shfl_xor_sync(0xffffffffu, bt, d);
      }
      double Ttot = __shfl_sync(0xffffffffu, incl, 31);
      bool direct = !(Ttot * p.kappa_max >= bt);  // cancellation (or NaN): take the direct tile totals
      int xsel = -1;
      bool ok = true;
      for (int attempt = 0; attempt < 2; ++attempt) {
        if (direct) {
          // tile totals from the panel rows themselves, in row order
          double sum = 0.0;
          const int x1 = min(L, (lane + 1) * Rt);
          // the tile's rows into L2 first (no registers held): the dependent batches below then
          // pay an L2 instead of a DRAM round trip each
          for (int x = lane * Rt; x < x1; x += 128 / (int)(sizeof(T) * B))
            asm volatile("prefetch.global.L2 [%0];" ::"l"(Ps + (size_t)x * B));
          for (int x = lane * Rt; x < x1; x += 4) {
            double w4[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int xx = min(x + j, L - 1);
              w4[j] = weight(xx);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (x + j < x1 && !masked(x + j)) sum += w4[j];
          }
          f = sum;
          incl = scan(f);
          Ttot = __shfl_sync(0xffffffffu, incl, 31);
          ++ndirect;
        }
        ok = (Ttot > 0.0) && (Ttot <= 1.7976931348623157e308);
        if (!ok) {
          if (direct) break;
          direct = true;
          continue;
        }
        const double thr = u * Ttot;
        const unsigned cross = __ballot_sync(0xffffffffu, f > 0.0 && incl > thr);
        const unsigned posl = __ballot_sync(0xffffffffu, f > 0.0);
        const int tau = cross ? __ffs(cross) - 1 : 31 - __clz(posl);  // posl != 0 since T > 0
        double ex = __shfl_up_sync(0xffffffffu, incl, 1);
        if (lane == 0) ex = 0.0;
        const double thr_in = thr - __shfl_sync(0xffffffffu, ex, tau);
        // ---- rows of tile tau, Rl consecutive rows per lane (row order = scan order)
        const int xb = tau * Rt + lane * Rl;
        double c[kGramMaxRl];
        double run = 0.0;
#pragma unroll
        for (int g4 = 0; g4 < kGramMaxRl; g4 += 4) {
          double w4[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int x = xb + g4 + j;
            w4[j] = (g4 + j < Rl) ? weight(min(x, L - 1)) : 0.0;
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int x = xb + g4 + j;
            const bool in = g4 + j < Rl && x < L;
            if (in && !masked(x)) run += w4[j];
            c[g4 + j] = run;
          }
        }
        const double incl2 = scan(run);
        double ex2 = __shfl_up_sync(0xffffffffu, incl2, 1);
        if (lane == 0) ex2 = 0.0;
        // the threshold inside the tile, as the same FRACTION of the tile's own row-wise total D
        // that thr_in is of the tile total f used by the tile scan (the two totals differ by
        // rounding); no crossing tile (u T >= T after rounding): the last row with w > 0
        const double Dt = __shfl_sync(0xffffffffu, incl2, 31);
        const double thr2 = cross ? (thr_in / __shfl_sync(0xffffffffu, f, tau)) * Dt : 1.7976931348623157e308;
        const double tp = thr2 - ex2;
        int rs = kGramMaxRl, rl = -1;
#pragma unroll
        for (int j = kGramMaxRl - 1; j >= 0; --j) {
          const double prev = j > 0 ? c[j - 1] : 0.0;
          if (c[j] > prev && c[j] > tp) rs = j;
        }
#pragma unroll
        for (int j = 0; j < kGramMaxRl; ++j) {
          const double prev = j > 0 ? c[j - 1] : 0.0;
          if (c[j] > prev) rl = j;
        }
        const unsigned b1 = __ballot_sync(0xffffffffu, rs < kGramMaxRl);
        if (b1) {
          const int ln = __ffs(b1) - 1;
          xsel = tau * Rt + ln * Rl + __shfl_sync(0xffffffffu, rs, ln);
        } else {
          const unsigned b2 = __ballot_sync(0xffffffffu, rl >= 0);
          if (b2) {
            const int ln = 31 - __clz(b2);
            xsel = tau * Rt + ln * Rl + __shfl_sync(0xffffffffu, rl, ln);
          }
        }
        if (xsel >= 0 || direct) break;
        direct = true;  // the Gram total of this tile was rounding noise: recompute directly
      }
      if (xsel < 0) {
        // T not finite / positive (flag bit0): the smallest site not drawn yet
        flag |= 1;
        const int nwords = (L + 31) >> 5;
        for (int wb = 0; wb < nwords && xsel < 0; wb += 32) {
          const int wi = wb + lane;
          uint32_t word = wi < nwords ? ch[wi] : 0xffffffffu;
          if (wi == nwords - 1 && (L & 31)) word |= 0xffffffffu << (L & 31);
#pragma unroll
          for (int q = 0; q < r; ++q)
            if ((xsv[q] >> 5) == wi) word |= 1u << (xsv[q] & 31);
          const unsigned bf = __ballot_sync(0xffffffffu, word != 0xffffffffu);
          if (bf) {
            const int ln = __ffs(bf) - 1;
            const uint32_t wsel = __shfl_sync(0xffffffffu, word, ln);
            xsel = (wb + ln) * 32 + (__ffs(~wsel) - 1);
          }
        }
      }
      FFS_CHECK(xsel >= 0 && xsel < L);
      if (traced) {
        const double inv = ok ? 1.0 / Ttot : 0.0;
        double* tr = p.trace + ((i - p.S0) * Np + k) * (int64_t)L;
        for (int x = lane; x < L; x += 32) tr[x] = masked(x) ? 0.0 : weight(x) * inv;
      }
      // ---- pivot row: the original panel row with the block's earlier eliminations applied
      if (lane < B * kD) reinterpret_cast<double*>(&sm.xrow[0])[lane] = reinterpret_cast<const double*>(Ps + (size_t)xsel * B)[lane];
      __syncwarp();
      T v[B];
#pragma unroll
      for (int cc = 0; cc < B; ++cc) v[cc] = sm.xrow[cc];
#pragma unroll
      for (int s = 0; s < r; ++s) {
        const T lm = S::mul(v[s], sm.Pinv[s]);
#pragma unroll
        for (int cc = s + 1; cc < B; ++cc) v[cc] = S::fms(lm, sm.Row[s][cc], v[cc]);
      }
      const T piv = v[r];
      if (ok && S::abs2(piv) < 1e-12 * Ttot) flag |= 2;
      const T ip = S::recip(piv);
      if (lane == 0) {
#pragma unroll
        for (int cc = 0; cc < B; ++cc) sm.Row[r][cc] = v[cc];
        sm.Pinv[r] = ip;
      }
      __syncwarp();
      // ---- Gauss-Jordan update of the in-block coefficients (lane = later column)
      if (lane > r && lane < B) {
        const T z = S::mul(sm.Row[r][lane], ip);
#pragma unroll
        for (int q = 0; q < r; ++q) sm.C[q][lane] = S::fms(sm.C[q][r], z, sm.C[q][lane]);
        sm.C[r][lane] = z;
      }
      __syncwarp();
      xsv[r] = xsel;
    }
  });

  // ---- hand S = L U of this block to the batched Gauss-Jordan kernel; positions, bitmap, flags
  T* rg = reinterpret_cast<T*>(p.rowg) + (size_t)sl * (B * B + B);
  for (int idx = lane; idx < B * B; idx += 32) rg[idx] = (&sm.Row[0][0])[idx];
  if (lane < B) rg[B * B + lane] = sm.Pinv[lane];
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < B; ++q)
      if (q < nb) {
        p.positions[i * Np + k0 + q] = xsv[q];
        atomicOr(ch + (xsv[q] >> 5), 1u << (xsv[q] & 31));
      }
    if (flag != 0 && p.flags != nullptr) atomicOr(reinterpret_cast<unsigned*>(p.flags + i), (unsigned)flag);
    if (p.stats != nullptr) {
      atomicAdd(p.stats, (unsigned long long)nb);
      if (ndirect) atomicAdd(p.stats + 1, (unsigned long long)ndirect);
    }
  }
}

}  // namespace ffsk
