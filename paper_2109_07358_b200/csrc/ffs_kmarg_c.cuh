// Tile-Gram marginal path for complex U (N' <= 32): the complex counterpart of ffs_kmarg.cuh's flat
// variant. With h' = (-A^{-1} V[X,k]; 1) and the bilinear s_k(x) = sum_q U[x, m_q] h'_q (reading Q3),
//   w_k(x) = |s_k(x)|^2,   sum_{x in tile} w_k(x) = h'^H K_tile[m, m] h',
//   K_tile[a][b] = sum_{x in tile} conj(U[x, a]) U[x, b]   (Hermitian, N x N),
// = sum_q |h_q|^2 K[q][q] + 2 Re sum_{q<q'} conj(h_q) h_q' K[q][q']. K is stored tile-minor,
// K[a][b][t] as (re, im) pairs, so a sample's read of one entry for all tiles is one coalesced row.
// One group of G lanes owns a sample, lane t evaluates tile t, exactly as in the real kernel; the
// coefficient matrix C = A^{-1} V[X, later columns] is complex and lives in shared memory.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ffs_kmarg.cuh"

namespace ffsk {

// K[a][b][t] = sum_{x in tile t} conj(U[x][a]) U[x][b]; grid (b tiles, a tiles, G), 256 threads,
// 32 x 32 outputs per CTA (2 x 2 per thread); a-tile <= b-tile computed, the conjugate mirror written
static __global__ void __launch_bounds__(256) ffs_tile_gram_uc_kernel(const double* __restrict__ U, double* __restrict__ K,
                                                                     int L, int N, int Rt, int G) {
  if (blockIdx.y > blockIdx.x) return;
  __shared__ double2 As[16][32 + 1], Bs[16][32 + 1];
  const double2* Uc = reinterpret_cast<const double2*>(U);
  const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
  const int a0 = blockIdx.y * 32, b0 = blockIdx.x * 32, tile = blockIdx.z;
  const int x0 = tile * Rt, x1 = min(L, x0 + Rt);
  double2 acc[2][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j] = make_double2(0.0, 0.0);
  for (int xc = x0; xc < x1; xc += 16) {
    __syncthreads();
    for (int idx = t; idx < 16 * 32; idx += 256) {
      const int k = idx >> 5, c = idx & 31, x = xc + k;
      As[k][c] = (x < x1 && a0 + c < N) ? Uc[(size_t)x * N + a0 + c] : make_double2(0.0, 0.0);
      Bs[k][c] = (x < x1 && b0 + c < N) ? Uc[(size_t)x * N + b0 + c] : make_double2(0.0, 0.0);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const double2 a = As[k][ty * 2 + i];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const double2 b = Bs[k][tx * 2 + j];
          acc[i][j].x = fma(a.x, b.x, fma(a.y, b.y, acc[i][j].x));    // conj(a) b
          acc[i][j].y = fma(a.x, b.y, fma(-a.y, b.x, acc[i][j].y));
        }
      }
    }
  }
  double2* Kt = reinterpret_cast<double2*>(K) + tile;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int a = a0 + ty * 2 + i, b = b0 + tx * 2 + j;
      if (a < N && b < N) {
        Kt[((size_t)a * N + b) * G] = acc[i][j];
        if (blockIdx.y != blockIdx.x) Kt[((size_t)b * N + a) * G] = make_double2(acc[i][j].x, -acc[i][j].y);
      }
    }
}

constexpr int kKmcMaxNp = 32;

// shared memory per sample owner: m, selection uniforms, d / U[x_k, m] / pivot row (complex), the
// entries' offsets in K and their complex coefficients, the drawn-row bitmap, C [N'][N'] complex
__host__ __device__ inline size_t kmargc_owner_smem(int L, int Np) {
  const size_t ne = ((size_t)Np * (Np + 1) / 2 + 15) & ~size_t(15);
  return align16(sizeof(int) * Np) + align16(sizeof(double) * Np) + 3 * align16(sizeof(cplx) * Np) +
         align16(sizeof(cplx) * ne) + align16(sizeof(int) * ne) + align16(sizeof(uint32_t) * ((L + 31) / 32)) +
         align16(sizeof(cplx) * Np * Np);
}

template <int RLMAX, int WARPS, int G>
static __global__ void __launch_bounds__(32 * WARPS) ffs_kmargc_kernel(const KMargParams p) {
  using S = Sc<cplx>;
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
  const size_t csz = align16(sizeof(cplx) * Np);
  int* m = reinterpret_cast<int*>(wb);
  double* uselv = reinterpret_cast<double*>(wb + align16(sizeof(int) * Np));
  cplx* dvec = reinterpret_cast<cplx*>(reinterpret_cast<unsigned char*>(uselv) + align16(sizeof(double) * Np));
  cplx* urow = reinterpret_cast<cplx*>(reinterpret_cast<unsigned char*>(dvec) + csz);
  cplx* vrow = reinterpret_cast<cplx*>(reinterpret_cast<unsigned char*>(urow) + csz);
  cplx* coef = reinterpret_cast<cplx*>(reinterpret_cast<unsigned char*>(vrow) + csz);
  int* koff = reinterpret_cast<int*>(reinterpret_cast<unsigned char*>(coef) + align16(sizeof(cplx) * ne_pad));
  uint32_t* bits = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(koff) + align16(sizeof(int) * ne_pad));
  cplx* C = reinterpret_cast<cplx*>(reinterpret_cast<unsigned char*>(bits) + align16(sizeof(uint32_t) * ((L + 31) / 32)));
  const int nwords = (L + 31) >> 5;
  const int64_t slot = ((int64_t)blockIdx.x * WARPS + warp) * NG + gi;
  const int64_t nslots = (int64_t)gridDim.x * WARPS * NG;
  const double2* Kl = reinterpret_cast<const double2*>(p.K) + lane;  // lane = tile
  const cplx* Ut = reinterpret_cast<const cplx*>(p.Ut);
  const cplx* Ug = reinterpret_cast<const cplx*>(p.U);
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
    for (int e = lane; e < ne_all; e += G) {
      const unsigned pr = pairs[e];
      koff[e] = (m[pr & 255u] * N + m[pr >> 8]) * G;  // K[m_q][m_q'], q <= q'
    }
    for (int e = ne_all + lane; e < ne_pad; e += G) koff[e] = 0;
    __syncwarp(gmask);
    int flag = 0;
    const bool traced = p.trace != nullptr && (uint64_t)(i - p.S0) < (uint64_t)p.S;

    for (int r = 0; r < Np; ++r) {
      const double u = uselv[r];
      const int mr = m[r];
      const int ne = (r + 1) * (r + 2) / 2;
      // ---- coefficients: diagonal |d_q|^2, pairs 2 conj(d_q) d_q' (q < q'); d = (dvec[0:r], 1)
      for (int qp = lane; qp <= r; qp += G) {
        const cplx dq = qp == r ? S::one() : dvec[qp];
        cplx* cc = coef + qp * (qp + 1) / 2;
        for (int q = 0; q < qp; ++q) {
          const cplx a = dvec[q];
          cc[q] = {2.0 * fma(a.re, dq.re, a.im * dq.im), 2.0 * fma(a.re, dq.im, -a.im * dq.re)};
        }
        cc[qp] = {S::abs2(dq), 0.0};
      }
      __syncwarp(gmask);
      // ---- tile totals f (lane = tile): sum Re(coef_e K_e)
      double f;
      {
        double a4[4] = {0.0, 0.0, 0.0, 0.0};
        const int ne8 = (ne + 7) & ~7;
        for (int e = lane + ne; e < ne8; e += G) coef[e] = {0.0, 0.0};
        __syncwarp(gmask);
        for (int e = 0; e < ne8; e += 8) {
          double2 g[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) g[j] = Kl[koff[e + j]];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const cplx c = coef[e + j];
            a4[j & 3] = fma(c.re, g[j].x, fma(-c.im, g[j].y, a4[j & 3]));
          }
        }
        f = (a4[0] + a4[1]) + (a4[2] + a4[3]);
      }
      if (f < 0.0) f = 0.0;

      auto srow = [&](int x) -> cplx {  // s(x) = sum_q U[x, m_q] d_q
        cplx sx = Ut[(size_t)mr * Lpt + x];
        for (int q = 0; q < r; ++q) sx = S::fms(Ut[(size_t)m[q] * Lpt + x], S::neg(dvec[q]), sx);
        return sx;
      };
      auto drawn = [&](int x) -> bool { return ((bits[x >> 5] >> (x & 31)) & 1u) != 0u; };

      double Ttot = 0.0;
      bool ok = true;
      int xsel = -1;
      for (int attempt = 0; attempt < 2; ++attempt) {
        if (attempt == 1) {  // the tile totals from the rows themselves (rare)
          double sum = 0.0;
          const int x1 = min(L, (lane + 1) * Rt);
          for (int x = lane * Rt; x < x1; ++x)
            if (!drawn(x)) sum += S::abs2(srow(x));
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
        // ---- rows of tile tau, Rl consecutive rows per lane, RLMAX at a time
        const int xb = (tau * G + lane) * Rl;
        auto chunk = [&](int c0, cplx (&s)[RLMAX]) {  // s(x) of rows xb + c0 .. (those < xb + Rl)
          const int nr = Rl - c0;
          // a full chunk of an even number of rows per lane: 32-byte loads (xb + c0 is even)
          const bool vec = RLMAX % 2 == 0 && nr >= RLMAX && (Rl & 1) == 0;
          auto ldcol = [&](const cplx* col, cplx (&dst)[RLMAX]) {
            if constexpr (RLMAX % 2 == 0) {
              if (vec) {
#pragma unroll
                for (int j = 0; j < RLMAX / 2; ++j)
                  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                      : "=d"(dst[2 * j].re), "=d"(dst[2 * j].im), "=d"(dst[2 * j + 1].re), "=d"(dst[2 * j + 1].im)
                      : "l"(col + 2 * j));
                return;
              }
            }
#pragma unroll
            for (int j = 0; j < RLMAX; ++j) dst[j] = j < nr ? col[j] : S::zero();
          };
          ldcol(Ut + (size_t)mr * Lpt + xb + c0, s);
          for (int q = 0; q < r; ++q) {
            const cplx dq = S::neg(dvec[q]);
            cplx cv[RLMAX];
            ldcol(Ut + (size_t)m[q] * Lpt + xb + c0, cv);
#pragma unroll
            for (int j = 0; j < RLMAX; ++j) s[j] = S::fms(cv[j], dq, s[j]);
          }
        };
        constexpr int kNoRow = 0x7fffffff;
        const bool one_chunk = RLMAX < 16 || Rl <= RLMAX;  // L <= G G RLMAX: the lane's prefix stays in registers
        double c[RLMAX];
        double run = 0.0;
        {
          cplx s[RLMAX];
          if constexpr (RLMAX < 16) {
            chunk(0, s);
#pragma unroll
            for (int j = 0; j < RLMAX; ++j) {
              const int x = xb + j;
              if (j < Rl && x < L && !drawn(x)) run += S::abs2(s[j]);
              c[j] = run;
            }
          } else {
            for (int c0 = 0; c0 < Rl; c0 += RLMAX) {
              chunk(c0, s);
#pragma unroll
              for (int j = 0; j < RLMAX; ++j) {
                const int x = xb + c0 + j;
                if (c0 + j < Rl && x < L && !drawn(x)) run += S::abs2(s[j]);
                c[j] = run;
              }
            }
          }
        }
        const double incl2 = scan(run);
        double ex2 = __shfl_up_sync(gmask, incl2, 1, G);
        if (lane == 0) ex2 = 0.0;
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
          cplx s[RLMAX];
          double pre = 0.0;
          for (int c0 = 0; c0 < Rl; c0 += RLMAX) {
            chunk(c0, s);
#pragma unroll
            for (int j = 0; j < RLMAX; ++j) {
              const int x = xb + c0 + j;
              if (c0 + j < Rl && x < L && !drawn(x)) {
                const double prev = pre;
                pre += S::abs2(s[j]);
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
      if (xsel < 0) {  // T not finite / positive (flag bit0): the smallest site not drawn yet
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
        for (int x = lane; x < L; x += G) tr[x] = drawn(x) ? 0.0 : S::abs2(srow(x)) * inv;
      }
      // ---- pivot row v[c] = V[x, c] - V[x, 0:r] C[0:r, c] (c >= r) and the Gauss-Jordan update
      for (int q = lane; q < Np; q += G) urow[q] = Ug[(size_t)xsel * N + m[q]];
      __syncwarp(gmask);
      for (int cc = r + lane; cc < Np; cc += G) {
        cplx a = urow[cc];
        for (int q = 0; q < r; ++q) a = S::fms(urow[q], C[(size_t)q * Np + cc], a);
        vrow[cc] = a;
      }
      __syncwarp(gmask);
      const cplx piv = vrow[r];
      if (ok && S::abs2(piv) < 1e-12 * Ttot) flag |= 2;
      const cplx ip = S::recip(piv);
      for (int cc = r + 1 + lane; cc < Np; cc += G) {
        const cplx z = S::mul(vrow[cc], ip);
        for (int q = 0; q < r; ++q) C[(size_t)q * Np + cc] = S::fms(C[(size_t)q * Np + r], z, C[(size_t)q * Np + cc]);
        C[(size_t)r * Np + cc] = z;
      }
      if (lane == 0) {
        bits[xsel >> 5] |= 1u << (xsel & 31);
        p.positions[i * Np + r] = xsel;
      }
      __syncwarp(gmask);
      if (r + 1 < Np)  // d of the next step: -(column r+1 of C)
        for (int q = lane; q <= r; q += G) dvec[q] = S::neg(C[(size_t)q * Np + r + 1]);
      __syncwarp(gmask);
    }
    if (lane == 0 && p.flags != nullptr) p.flags[i] = flag;
  }
}

}  // namespace ffsk
