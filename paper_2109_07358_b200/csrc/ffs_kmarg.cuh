// Tile-Gram marginal path: real U, small N' (marginals), any L.
//
// Step k of a sample has the weights w_k(x) = |u_x^T h'|^2 with h' = (-A^{-1} V[X,k]; 1) on the
// permuted columns m_0..m_k (Eq. 3), i.e. w_k(x) = (sum_{q<=k}
// U[x, m_q] d_q)^2 with d = h'. The total of w_k over a TILE of rows is the quadratic form
//   sum_{x in tile} w_k(x) = d^T K_tile[m, m] d,     K_tile = U_tile^T U_tile  (N x N),
// and K_tile does not depend on the sample: it is computed ONCE per call for 32 row tiles
// (ffs_tile_gram_u_kernel, L N^2 / 2 FMAs in all), after which a sample's step costs 32 forms of
// (k+1)(k+2)/2 terms plus the rows of the one tile the threshold u T falls in -- O(32 N'^3 / 6 +
// N'^2 L / 64) per sample instead of L N'^2 / 2. One warp owns a sample: lane t evaluates tile t,
// a warp scan finds the crossing tile, its L/32 rows are scanned for x_k, and the coefficient
// matrix C = A^{-1} V[X, later columns] takes a rank-1 Gauss-Jordan update. K is stored TILE-MINOR,
// K[a][b][t]: the 32 tile values of one entry are 256 contiguous bytes, so the warp's read of a
// sample's entry K_t[m_q][m_q'] (lane = t) is one coalesced row, straight from the shared K -- no
// per-sample copy of the gathered Gram matrix is kept (measured: gathering it into a per-warp
// slot cost 20 % of the instructions and wrote 35 KB per C3 sample back to DRAM).
// Conditioning: sum_t K_t = U^T U = 1, so by Cauchy-Schwarz sum_t |d^T K_t d| terms are bounded by
// (k+1) |d|^2 = (k+1) T: the forms never cancel by more than a factor N' (no guard needed).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ffs_kernel.cuh"

namespace ffsk {

// K[a][b][t] = sum_{x in tile t} U[x][a] U[x][b], G tiles of Rt rows; grid (b tiles, a tiles, G),
// 256 threads, 64 x 64 outputs per CTA (4 x 4 per thread); only a-tile <= b-tile is computed, the
// mirror image is written with it
static __global__ void __launch_bounds__(256) ffs_tile_gram_u_kernel(const double* __restrict__ U, double* __restrict__ K,
                                                                    int L, int N, int Rt, int G) {
  if (blockIdx.y > blockIdx.x) return;
  __shared__ double As[16][64 + 4], Bs[16][64 + 4];
  const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
  const int a0 = blockIdx.y * 64, b0 = blockIdx.x * 64, tile = blockIdx.z;
  const int x0 = tile * Rt, x1 = min(L, x0 + Rt);
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int xc = x0; xc < x1; xc += 16) {
    __syncthreads();
    for (int idx = t; idx < 16 * 64; idx += 256) {
      const int k = idx >> 6, c = idx & 63, x = xc + k;
      As[k][c] = (x < x1 && a0 + c < N) ? U[(size_t)x * N + a0 + c] : 0.0;
      Bs[k][c] = (x < x1 && b0 + c < N) ? U[(size_t)x * N + b0 + c] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[k][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[k][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
  }
  double* Kt = K + tile;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int a = a0 + ty * 4 + i, b = b0 + tx * 4 + j;
      if (a < N && b < N) {
        Kt[((size_t)a * N + b) * G] = acc[i][j];
        if (blockIdx.y != blockIdx.x) Kt[((size_t)b * N + a) * G] = acc[i][j];
      }
    }
}

struct KMargParams {
  const double* U;         // [L][N]
  const double* Ut;        // [N][Lpt] transposed, zero-padded, Lpt = G G Rl
  const double* K;         // [N][N][G] tile Gram matrices of U, tile-minor
  const int32_t* permg;    // [M][Np]
  const double* uniforms;  // [M][2Np]
  int32_t* positions;      // [M][Np]
  int32_t* flags;          // [M] or null
  double* Cw;              // [slots][Np][Np] coefficient matrix (null: in shared memory)
  int L, N, Np, Lpt, Rl;   // Rl rows per lane of a tile (tile = G Rl rows, G tiles; G = lanes per sample)
  int64_t M, S0, S;
  double* trace;           // [S][Np][L] or null
  size_t warp_smem;        // bytes of shared memory per sample owner (a group of G lanes)
  double kappa_max;        // blocked forms: cancellation guard (as ffs_gram.cuh)
};

constexpr int kKmMaxNp = 96;

// shared memory per sample owner (a warp, or a half warp when L <= 1024: G = 16 lanes, 16 tiles): m, selection uniforms, d, U[x_k, m], pivot row, the drawn-row bitmap,
// (small N') C, and for the forms either the offsets of the sample's entries in K + their
// coefficients (flat evaluation), or the block's D, tile Gram entries and their sqrt-diagonal
// (blocked evaluation)
__host__ __device__ inline size_t kmarg_warp_smem(int L, int Np, bool c_smem, bool blocked, int G) {
  const size_t ne = ((size_t)Np * (Np + 1) / 2 + 15) & ~size_t(15);  // padded to the form's batch of 16
  const size_t forms = blocked ? sizeof(double) * (48 + (size_t)Np * 8 + 36 * G + 8 * G)
                               : align16(sizeof(double) * ne) + align16(sizeof(int) * ne);
  return align16(sizeof(int) * Np) + 4 * align16(sizeof(double) * Np) + forms +
         align16(sizeof(uint32_t) * ((L + 31) / 32)) + (c_smem ? align16(sizeof(double) * Np * Np) : 0);
}

// G lanes own a sample (G = 32: a warp; G = 16: a half warp, two samples per warp -- for small L the
// per-draw work is dominated by steps that keep <= 16 lanes busy). `lane` below is the lane WITHIN
// the owner group; every shuffle / ballot / barrier is restricted to the group's lanes.
template <int RLMAX, int WARPS, bool BLK, int G>
static __global__ void __launch_bounds__(32 * WARPS, (RLMAX <= 4 && !BLK) ? 6 : 1) ffs_kmarg_kernel(const KMargParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int NG = 32 / G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & (G - 1), gi = (threadIdx.x & 31) / G;
  const unsigned gmask = G == 32 ? 0xffffffffu : (0xffffu << (16 * gi));
  auto gballot = [&](bool pred) -> unsigned {
    const unsigned bsel = __ballot_sync(gmask, pred);
    return G == 32 ? bsel : ((bsel >> (16 * gi)) & 0xffffu);
  };
  const int L = p.L, N = p.N, Np = p.Np, Rl = p.Rl, Lpt = p.Lpt;
  const int Rt = G * Rl;
  const int ne_all = Np * (Np + 1) / 2;
  const int ne_pad = (ne_all + 15) & ~15;
  unsigned char* wb = smem + (size_t)(warp * NG + gi) * p.warp_smem;
  const size_t dsz = align16(sizeof(double) * Np);
  int* m = reinterpret_cast<int*>(wb);
  double* uselv = reinterpret_cast<double*>(wb + align16(sizeof(int) * Np));
  double* dvec = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(uselv) + dsz);
  double* urow = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(dvec) + dsz);
  double* vrow = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(urow) + dsz);
  double* coef = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(vrow) + dsz);
  // flat: coef [ne_pad], koff [ne_pad]; blocked: coef [48], Dm [Np][8], gbs [36][32], sgs [8][32]
  int* koff = reinterpret_cast<int*>(reinterpret_cast<unsigned char*>(coef) + align16(sizeof(double) * ne_pad));
  double* Dm = coef + 48;
  double* gbs = Dm + (size_t)Np * 8;
  double* sgs = gbs + 36 * G;
  uint32_t* bits = BLK ? reinterpret_cast<uint32_t*>(sgs + 8 * G)
                       : reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(koff) + align16(sizeof(int) * ne_pad));
  unsigned char* extra = reinterpret_cast<unsigned char*>(bits) + align16(sizeof(uint32_t) * ((L + 31) / 32));
  const int nwords = (L + 31) >> 5;
  const int64_t slot = ((int64_t)blockIdx.x * WARPS + warp) * NG + gi;
  const int64_t nslots = (int64_t)gridDim.x * WARPS * NG;
  double* C = p.Cw != nullptr ? p.Cw + (size_t)slot * Np * Np : reinterpret_cast<double*>(extra);
  const double* Kl = p.K + lane;  // lane = tile
  // entry e <-> (q, q'), q <= q', e = q'(q'+1)/2 + q: one table per CTA
  uint16_t* pairs = reinterpret_cast<uint16_t*>(smem + (size_t)WARPS * NG * p.warp_smem);
  for (int e = threadIdx.x; e < ne_all; e += blockDim.x) {
    int qp = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
    while ((qp + 1) * (qp + 2) / 2 <= e) ++qp;
    while (qp * (qp + 1) / 2 > e) --qp;
    pairs[e] = (uint16_t)((e - qp * (qp + 1) / 2) | (qp << 8));
  }
  __syncthreads();

  auto scan = [&](double v) -> double {
#pragma unroll
    for (int d = 1; d < G; d <<= 1) {
      const double y = __shfl_up_sync(gmask, v, d, G);
      if (lane >= d) v += y;
    }
    return v;
  };

  for (int64_t i = slot; i < p.M; i += nslots) {
    __syncwarp(gmask);
    for (int j = lane; j < Np; j += G) {
      m[j] = p.permg[i * Np + j];
      FFS_CHECK(m[j] >= 0 && m[j] < N);
      uselv[j] = p.uniforms[i * 2 * (int64_t)Np + Np + j];
    }
    for (int j = lane; j < nwords; j += G) bits[j] = 0u;
    __syncwarp(gmask);
    // ---- offsets of the sample's Gram entries G[q][q'] = K[m_q][m_q'][:] in K (entry e by lane e mod 32)
    if constexpr (!BLK) {
      for (int e = lane; e < ne_all; e += G) {
        const unsigned pr = pairs[e];
        koff[e] = (m[pr & 255u] * N + m[pr >> 8]) * G;
      }
      for (int e = ne_all + lane; e < ne_pad; e += G) koff[e] = 0;
      __syncwarp(gmask);
    }
    int flag = 0;
    const bool traced = p.trace != nullptr && (uint64_t)(i - p.S0) < (uint64_t)p.S;

    for (int r = 0; r < Np; ++r) {
      const double u = uselv[r];
      const int mr = m[r];
      const int ne = (r + 1) * (r + 2) / 2;
      double f = 0.0;
      if constexpr (BLK) {
        // ---- blocked evaluation: at a block start k0 the tile Gram matrix of the block's 8 Schur
        // columns, G_blk = D^T G D with D = (-C[0:k0, k0:k0+8]; I) -- every entry of
        // G[0:k0+8, 0:k0+8] is read once per BLOCK; the draws of the block then use 36-term forms
        // with the in-block coefficients d_blk = (-C[k0:k, k]; 1)
        const int rb = r & 7, k0 = r - rb;
        if (rb == 0) {
          const int nb = min(8, Np - k0), na = k0 + nb;
          for (int idx = lane; idx < na * 8; idx += G) {
            const int a = idx >> 3, c = idx & 7;
            Dm[idx] = a < k0 ? (c < nb ? -C[(size_t)a * Np + k0 + c] : 0.0) : (a - k0 == c ? 1.0 : 0.0);
          }
          __syncwarp(gmask);
          double gb[36];
#pragma unroll
          for (int e = 0; e < 36; ++e) gb[e] = 0.0;
          for (int a = 0; a < na; a += 2) {
            const int a1 = min(a + 1, na - 1);
            const double* Ka = Kl + (size_t)m[a] * N * G;
            const double* Kb = Kl + (size_t)m[a1] * N * G;
            double t0[8], t1[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) t0[c] = t1[c] = 0.0;
            for (int b = 0; b < na; b += 8) {
              double g0[8], g1[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const int mb = m[min(b + j, na - 1)] * G;
                g0[j] = Ka[mb];
                g1[j] = Kb[mb];
              }
#pragma unroll
              for (int j = 0; j < 8; ++j)
                if (b + j < na) {
                  const double2* dr = reinterpret_cast<const double2*>(Dm + (size_t)(b + j) * 8);
#pragma unroll
                  for (int c2 = 0; c2 < 4; ++c2) {
                    const double2 d2 = dr[c2];
                    t0[2 * c2] = fma(g0[j], d2.x, t0[2 * c2]);
                    t0[2 * c2 + 1] = fma(g0[j], d2.y, t0[2 * c2 + 1]);
                    t1[2 * c2] = fma(g1[j], d2.x, t1[2 * c2]);
                    t1[2 * c2 + 1] = fma(g1[j], d2.y, t1[2 * c2 + 1]);
                  }
                }
            }
            const double* da = Dm + (size_t)a * 8;
            const double* db = Dm + (size_t)a1 * 8;
            const bool two = a + 1 < na;
#pragma unroll
            for (int c1 = 0; c1 < 8; ++c1)
#pragma unroll
              for (int c = 0; c <= c1; ++c) {
                gb[c1 * (c1 + 1) / 2 + c] = fma(da[c], t0[c1], gb[c1 * (c1 + 1) / 2 + c]);
                if (two) gb[c1 * (c1 + 1) / 2 + c] = fma(db[c], t1[c1], gb[c1 * (c1 + 1) / 2 + c]);
              }
          }
#pragma unroll
          for (int e = 0; e < 36; ++e) gbs[e * G + lane] = gb[e];
#pragma unroll
          for (int q = 0; q < 8; ++q) sgs[q * G + lane] = sqrt(fmax(gb[q * (q + 1) / 2 + q], 0.0));
        }
        if (lane <= rb) {
          const int qp = lane;
          const double dq = qp == rb ? 1.0 : dvec[k0 + qp];
          double* cc = coef + qp * (qp + 1) / 2;
          for (int q = 0; q < qp; ++q) cc[q] = 2.0 * dq * dvec[k0 + q];
          cc[qp] = dq * dq;
        }
        __syncwarp(gmask);
        const int neb = (rb + 1) * (rb + 2) / 2;
        for (int e = 0; e < neb; ++e) f = fma(coef[e], gbs[e * G + lane], f);
        // cancellation guard (as ffs_gram.cuh): bound (sum_q |d_q| sqrt(G_blk[q][q]))^2 against the total
        double bd = sgs[rb * G + lane];
        for (int q = 0; q < rb; ++q) bd = fma(fabs(dvec[k0 + q]), sgs[q * G + lane], bd);
        bd *= bd;
        double ft = f > 0.0 ? f : 0.0;
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {
          ft += __shfl_xor_sync(gmask, ft, o, G);
          bd += __shfl_xor_sync(gmask, bd, o, G);
        }
        if (!(ft * p.kappa_max >= bd)) {
          // rare: the form on the ORIGINAL columns (conditioned within a factor N'), entry by entry
          f = 0.0;
          for (int qp = 0; qp <= r; ++qp) {
            const double dq = qp == r ? 1.0 : dvec[qp];
            const double* Kc = Kl + (size_t)m[qp] * G;
            double acc = 0.0;
            for (int q = 0; q < qp; ++q) acc = fma(Kc[(size_t)m[q] * N * G], dvec[q], acc);
            f = fma(dq, fma(Kc[(size_t)m[qp] * N * G], dq, 2.0 * acc), f);
          }
        }
      } else {
        // ---- coefficients of the form d^T G d, d = (dvec[0:r], 1): column q' by lane q' (mod 32)
        for (int qp = lane; qp <= r; qp += G) {
          const double dq = qp == r ? 1.0 : dvec[qp];
          double* cc = coef + qp * (qp + 1) / 2;
          for (int q = 0; q < qp; ++q) cc[q] = 2.0 * dq * dvec[q];
          cc[qp] = dq * dq;
        }
        __syncwarp(gmask);
        // ---- tile totals f (lane = tile)
        {
          double a[8];
  #pragma unroll
          for (int j = 0; j < 8; ++j) a[j] = 0.0;
          // batches of 16 entries: offsets and coefficients by 16-byte broadcast reads, the 16 K rows
          // in flight together (the arrays are padded to a multiple of 16 entries: coefficient 0)
          const int ne16 = (ne + 15) & ~15;
          for (int e = lane + ne; e < ne16; e += G) coef[e] = 0.0;
          __syncwarp(gmask);
          for (int e = 0; e < ne16; e += 16) {
            int ko[16];
            double g[16], cf[16];
  #pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int4 k4 = *reinterpret_cast<const int4*>(koff + e + 4 * j);
              ko[4 * j] = k4.x;
              ko[4 * j + 1] = k4.y;
              ko[4 * j + 2] = k4.z;
              ko[4 * j + 3] = k4.w;
            }
  #pragma unroll
            for (int j = 0; j < 16; ++j) g[j] = Kl[ko[j]];
  #pragma unroll
            for (int j = 0; j < 8; ++j) {
              const double2 c2 = *reinterpret_cast<const double2*>(coef + e + 2 * j);
              cf[2 * j] = c2.x;
              cf[2 * j + 1] = c2.y;
            }
  #pragma unroll
            for (int j = 0; j < 16; ++j) a[j & 7] = fma(g[j], cf[j], a[j & 7]);
          }
          f = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
        }
      }
      if (f < 0.0) f = 0.0;

      // s(x) = sum_q U[x, m_q] d_q for one row (fallbacks, trace)
      auto srow = [&](int x) -> double {
        double sx = p.Ut[(size_t)mr * Lpt + x];
        for (int q = 0; q < r; ++q) sx = fma(p.Ut[(size_t)m[q] * Lpt + x], dvec[q], sx);
        return sx;
      };
      auto drawn = [&](int x) -> bool { return ((bits[x >> 5] >> (x & 31)) & 1u) != 0u; };

      double Ttot = 0.0;
      bool ok = true;
      int xsel = -1;
      for (int attempt = 0; attempt < 2; ++attempt) {
        if (attempt == 1) {
          // the tile totals from the rows themselves (the form of a tile was rounding noise, or T
          // is degenerate): rare
          double sum = 0.0;
          const int x1 = min(L, (lane + 1) * Rt);
          for (int x = lane * Rt; x < x1; ++x)
            if (!drawn(x)) {
              const double sx = srow(x);
              sum = fma(sx, sx, sum);
            }
          f = sum;
        }
        const double incl = scan(f);
        Ttot = __shfl_sync(gmask, incl, G - 1, G);
        ok = (Ttot > 0.0) && (Ttot <= 1.7976931348623157e308);
        if (!ok) continue;
        const double thr = u * Ttot;
        const unsigned cross = gballot(f > 0.0 && incl > thr);
        const unsigned posl = gballot(f > 0.0);
        const int tau = cross ? __ffs(cross) - 1 : 31 - __clz(posl);
        double ex = __shfl_up_sync(gmask, incl, 1, G);
        if (lane == 0) ex = 0.0;
        const double thr_in = thr - __shfl_sync(gmask, ex, tau, G);
        // ---- rows of tile tau, Rl consecutive rows per lane, RLMAX at a time: s(x) = sum_q U[x, m_q] d_q
        const int xb = (tau * G + lane) * Rl;
        auto chunk = [&](int c0, double (&s)[RLMAX]) {  // rows xb + c0 .. xb + c0 + RLMAX - 1 (those < xb + Rl)
          const int nr = Rl - c0;
          // a full chunk of an even number of rows per lane: 16-byte loads (xb + c0 is even)
          const bool vec = RLMAX % 2 == 0 && nr >= RLMAX && (Rl & 1) == 0;
          auto ldcol = [&](const double* col, double (&dst)[RLMAX]) {
            if constexpr (RLMAX % 4 == 0) {
              if (vec && (Rl & 3) == 0) {  // 32-byte loads
#pragma unroll
                for (int j = 0; j < RLMAX / 4; ++j)
                  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                      : "=d"(dst[4 * j]), "=d"(dst[4 * j + 1]), "=d"(dst[4 * j + 2]), "=d"(dst[4 * j + 3])
                      : "l"(col + 4 * j));
                return;
              }
            }
            if constexpr (RLMAX % 2 == 0) {
              if (vec) {
#pragma unroll
                for (int j = 0; j < RLMAX / 2; ++j) {
                  const double2 v = reinterpret_cast<const double2*>(col)[j];
                  dst[2 * j] = v.x;
                  dst[2 * j + 1] = v.y;
                }
                return;
              }
            }
#pragma unroll
            for (int j = 0; j < RLMAX; ++j) dst[j] = j < nr ? col[j] : 0.0;
          };
          ldcol(p.Ut + (size_t)mr * Lpt + xb + c0, s);
          constexpr int QB = RLMAX == 1 ? 8 : RLMAX <= 4 ? 4 : 2;  // columns in flight
          int q = 0;
          for (; q + QB <= r; q += QB) {
            double cv[QB][RLMAX];
#pragma unroll
            for (int b = 0; b < QB; ++b) ldcol(p.Ut + (size_t)m[q + b] * Lpt + xb + c0, cv[b]);
#pragma unroll
            for (int b = 0; b < QB; ++b) {
              const double dq = dvec[q + b];
#pragma unroll
              for (int j = 0; j < RLMAX; ++j) s[j] = fma(cv[b][j], dq, s[j]);
            }
          }
          for (; q < r; ++q) {
            const double dq = dvec[q];
            const double* col = p.Ut + (size_t)m[q] * Lpt + xb + c0;
#pragma unroll
            for (int j = 0; j < RLMAX; ++j)
              if (j < nr) s[j] = fma(col[j], dq, s[j]);
          }
        };
        constexpr int kNoRow = 0x7fffffff;
        // L <= G G RLMAX (always for RLMAX < 16): the prefix of the lane's rows stays in registers
        const bool one_chunk = RLMAX < 16 || Rl <= RLMAX;
        double c[RLMAX];
        double run = 0.0;
        {
          double s[RLMAX];
          if constexpr (RLMAX < 16) {
            chunk(0, s);
#pragma unroll
            for (int j = 0; j < RLMAX; ++j) {
              const int x = xb + j;
              if (j < Rl && x < L && !drawn(x)) run = fma(s[j], s[j], run);
              c[j] = run;
            }
          } else {
            for (int c0 = 0; c0 < Rl; c0 += RLMAX) {
              chunk(c0, s);
#pragma unroll
              for (int j = 0; j < RLMAX; ++j) {
                const int x = xb + c0 + j;
                if (c0 + j < Rl && x < L && !drawn(x)) run = fma(s[j], s[j], run);
                c[j] = run;
              }
            }
          }
        }
        const double incl2 = scan(run);
        double ex2 = __shfl_up_sync(gmask, incl2, 1, G);
        if (lane == 0) ex2 = 0.0;
        // the in-tile threshold as the same fraction of the tile's row-wise total that thr_in is
        // of the tile total used by the tile scan (they differ by rounding); u T >= T after
        // rounding: the last row with w > 0
        const double Dt = __shfl_sync(gmask, incl2, G - 1, G);
        const double thr2 = cross ? (thr_in / __shfl_sync(gmask, f, tau, G)) * Dt : 1.7976931348623157e308;
        const double tp = thr2 - ex2;
        int rs = kNoRow, rl = -1;  // first row of this lane past the threshold / its last row with w > 0
        if (one_chunk) {
#pragma unroll
          for (int j = RLMAX - 1; j >= 0; --j) {
            const double prev = j > 0 ? c[j - 1] : 0.0;
            if (c[j] > prev && c[j] > tp) rs = j;
          }
#pragma unroll
          for (int j = 0; j < RLMAX; ++j) {
            const double prev = j > 0 ? c[j - 1] : 0.0;
            if (c[j] > prev) rl = j;
          }
        } else if constexpr (RLMAX >= 16) {
          // large L: the same sums again, chunk by chunk (identical order, so the last prefix is `run`)
          double s[RLMAX];
          double pre = 0.0;
          for (int c0 = 0; c0 < Rl; c0 += RLMAX) {
            chunk(c0, s);
#pragma unroll
            for (int j = 0; j < RLMAX; ++j) {
              const int x = xb + c0 + j;
              if (c0 + j < Rl && x < L && !drawn(x)) {
                const double prev = pre;
                pre = fma(s[j], s[j], pre);
                if (pre > prev) {
                  rl = c0 + j;
                  if (rs == kNoRow && pre > tp) rs = c0 + j;
                }
              }
            }
          }
        }
        const unsigned b1 = gballot(rs != kNoRow);
        if (b1) {
          const int ln = __ffs(b1) - 1;
          xsel = (tau * G + ln) * Rl + __shfl_sync(gmask, rs, ln, G);
        } else {
          const unsigned b2 = gballot(rl >= 0);
          if (b2) {
            const int ln = 31 - __clz(b2);
            xsel = (tau * G + ln) * Rl + __shfl_sync(gmask, rl, ln, G);
          }
        }
        if (xsel >= 0) break;
      }
      if (xsel < 0) {
        // T not finite / positive (flag bit0): the smallest site not drawn yet
        flag |= 1;
        for (int wbase = 0; wbase < nwords && xsel < 0; wbase += G) {
          const int wi = wbase + lane;
          uint32_t word = wi < nwords ? bits[wi] : 0xffffffffu;
          if (wi == nwords - 1 && (L & 31)) word |= 0xffffffffu << (L & 31);
          const unsigned bf = gballot(word != 0xffffffffu);
          if (bf) {
            const int ln = __ffs(bf) - 1;
            const uint32_t wsel = __shfl_sync(gmask, word, ln, G);
            xsel = (wbase + ln) * 32 + (__ffs(~wsel) - 1);
          }
        }
      }
      FFS_CHECK(xsel >= 0 && xsel < L);
      if (traced) {
        const double inv = ok ? 1.0 / Ttot : 0.0;
        double* tr = p.trace + ((i - p.S0) * Np + r) * (int64_t)L;
        for (int x = lane; x < L; x += G) {
          const double sx = srow(x);
          tr[x] = drawn(x) ? 0.0 : sx * sx * inv;
        }
      }
      // ---- pivot row v[c] = V[x, c] - V[x, 0:r] C[0:r, c] (c >= r) and the Gauss-Jordan update
      for (int q = lane; q < Np; q += G) urow[q] = p.U[(size_t)xsel * N + m[q]];
      __syncwarp(gmask);
      for (int cc = r + lane; cc < Np; cc += G) {
        double a0 = urow[cc], a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int q = 0;
        for (; q + 4 <= r; q += 4) {
          const double w0 = C[(size_t)q * Np + cc], w1 = C[(size_t)(q + 1) * Np + cc];
          const double w2 = C[(size_t)(q + 2) * Np + cc], w3 = C[(size_t)(q + 3) * Np + cc];
          a0 = fma(-urow[q], w0, a0);
          a1 = fma(-urow[q + 1], w1, a1);
          a2 = fma(-urow[q + 2], w2, a2);
          a3 = fma(-urow[q + 3], w3, a3);
        }
        for (; q < r; ++q) a0 = fma(-urow[q], C[(size_t)q * Np + cc], a0);
        vrow[cc] = (a0 + a1) + (a2 + a3);
      }
      __syncwarp(gmask);
      const double piv = vrow[r];
      if (ok && piv * piv < 1e-12 * Ttot) flag |= 2;
      const double ip = fast_rcp(piv);
      for (int cc = r + 1 + lane; cc < Np; cc += G) {
        const double z = vrow[cc] * ip;
        int q = 0;
        for (; q + 4 <= r; q += 4) {
          double w[4], cr[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            w[j] = C[(size_t)(q + j) * Np + cc];
            cr[j] = C[(size_t)(q + j) * Np + r];
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) C[(size_t)(q + j) * Np + cc] = fma(-cr[j], z, w[j]);
        }
        for (; q < r; ++q) C[(size_t)q * Np + cc] = fma(-C[(size_t)q * Np + r], z, C[(size_t)q * Np + cc]);
        C[(size_t)r * Np + cc] = z;
      }
      if (lane == 0) {
        bits[xsel >> 5] |= 1u << (xsel & 31);
        p.positions[i * Np + r] = xsel;
      }
      __syncwarp(gmask);
      // d of the next step: -(column r+1 of C)
      if (r + 1 < Np)
        for (int q = lane; q <= r; q += G) dvec[q] = -C[(size_t)q * Np + r + 1];
      __syncwarp(gmask);
    }
    if (lane == 0 && p.flags != nullptr) p.flags[i] = flag;
  }
}

}  // namespace ffsk
