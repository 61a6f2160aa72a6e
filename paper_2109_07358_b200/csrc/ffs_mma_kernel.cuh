// Warp-owner FFS kernel with the panel contraction on the FP64 tensor path (DMMA m8n8k4), for
// real U with 128 < L <= 256 and N' <= kMaxNpWarp: the headline double-well workload (C2).
//
// Same mathematics as ffs_seg_kernel (blocked left-looking randomized-pivot LU):
//   a3  P = V[:, k0:k0+8] - V[:, 0:k0] W[0:k0, k0:k0+8]     (per-sample gathered V = U[:, m])
//   a4  8 sequential draws on the register panel (weights |P[:,r]|^2, warp scan, inverse CDF)
//   a5  rank-1 updates of the later panel columns; Gauss-Jordan update of W = A^{-1} V[X, later]
// What changes is how a3 is issued. With a panel of B = 8 columns the contraction of one sample is
// an (L x k0) x (k0 x 8) product whose A operand is gathered per sample; it maps onto
// mma.sync.m8n8k4.f64 with M = 8 rows x of U, N = the 8 panel columns, K = 4 permuted columns:
// one DMMA (256 FMA) replaces eight warp-wide DFMA and their operand loads, which frees the issue
// slots and shared-memory wavefronts that bound the DFMA formulation (profiles/r01_ncu_summary.md).
// The FP64 pipe does the same FMA work either way (DMMA and DFMA share it on B200).
//
// Layouts
//   * U^T in shared memory, 256 rows per column (rows >= L zero). Row x is element x&1 of the
//     16-byte chunk q = x>>1; chunks are stored 128-byte-line swizzled: line = q>>3, slot = (q&7) ^
//     (line&7). Every warp-wide access pattern below (A fragments, accumulator init, Gauss-Jordan
//     gathers) then touches each bank at most the minimum number of times.
//   * MMA layout of the contraction: lane (g = lane>>2, t4 = lane&3); tile pair pi = 4j + a
//     (j, a in 0..3), tile e in {0,1}; MMA row g of tile (pi, e) is the row x = 64a + 8g + 2j + e, so
//     one LDS.128 fetches the A elements of both tiles of a pair. Accumulator acc[pi][e][h] is
//     P[x][2 t4 + h].
//   * draw layout (as ffs_seg_kernel, R = 8): lane l owns rows 8l .. 8l+7 of all 8 columns,
//     P[r][c]. Row x = 64a + 8g + 2j + e lands in lane 8a + g, row slot 2j + e: round j of the
//     transposition moves rows 2j, 2j+1 of every lane through a 4 KB per-warp shared buffer
//     (16-byte chunks swizzled by (lane & 7): conflict-free stores and loads).
//   * per-owner slice (WarpLayout-like, see MmaLayout): permutation (U^T column offsets),
//     positions, selection uniforms, pivot rows (B x B), inverse pivots, W [N'][ldw], and the
//     transposition buffer, which the Gauss-Jordan update reuses for VnT.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ffs_warp_kernel.cuh"

namespace ffsk {

constexpr int kMmaRows = 256;  // U^T column length in shared memory (L <= 256)

struct MmaLayout {
  size_t perm, pos, usel, row, pinv, wf, buf, total;
  int ldw;
  __host__ __device__ explicit MmaLayout(int Np) {
    constexpr int B = 8;
    // W row stride: N'+2 when 8 | N' (rows 16 B apart in bank space); otherwise room for the
    // zero columns the ragged last block reads
    ldw = (Np % B == 0) ? ((Np + 3) & ~1) : ((Np + B + 1) & ~1);
    size_t o = 0;
    perm = o; o = align16(o + sizeof(int) * Np);
    pos = o;  o = align16(o + sizeof(int) * Np);
    usel = o; o = align16(o + sizeof(double) * Np);
    row = o;  o = align16(o + sizeof(double) * B * B);
    pinv = o; o = align16(o + sizeof(double) * B);
    wf = o;   o = align16(o + sizeof(double) * (size_t)Np * ldw);
    const size_t vnt = sizeof(double) * (size_t)Np * B;
    const size_t tb = sizeof(double) * 32 * 16;  // transposition buffer: 32 lanes x 16 doubles
    buf = o;  o = align16(o + (vnt > tb ? vnt : tb));
    total = o;
  }
};

// element index of row x inside a U^T column (swizzled 16-byte chunks, see the header)
__host__ __device__ __forceinline__ int mma_phys(int x) {
  const int q = x >> 1, line = q >> 3;
  return (((line << 3) | ((q & 7) ^ (line & 7))) << 1) | (x & 1);
}

// D = A B + D, m8n8k4, fp64 (DMMA.8x8x4 on sm_100a)
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Gauss-Jordan update of one owner's W with the B = 8 new rows (see seg_gj_flat; only the U^T
// swizzle differs).
__device__ __forceinline__ void mma_gj(const double* __restrict__ Uts, const int* perm, const int* pos,
                                       const double* Row, const double* Pinv, double* Wf, double* VnT, int ldw,
                                       int k0, int Np, int sl) {
  constexpr int B = 8, G = 32;
  const int j0 = k0 + B, nc = Np - j0;
  __syncwarp();
  {
    const int t = sl % B;
    const int xp = mma_phys(pos[k0 + t]);
    for (int idx = sl; idx < Np * B; idx += G) VnT[idx] = Uts[perm[idx / B] + xp];
  }
  __syncwarp();
  for (int idx = sl; idx < nc * B; idx += G) {
    const int t = idx % B, j = j0 + idx / B;
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

template <int MAXT>
__global__ void __launch_bounds__(MAXT, 1) ffs_mma_kernel(const WarpParams p) {
  constexpr int R = 8, B = 8, G = 32;
  extern __shared__ __align__(16) unsigned char smem[];  // dynamic smem base is 1 KB aligned
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int L = p.L, N = p.N, Np = p.Np;

  // ---- U^T into shared memory (swizzled; rows >= L zero)
  double* Uts = reinterpret_cast<double*>(smem);
  for (int idx = threadIdx.x; idx < N * kMmaRows; idx += blockDim.x) {
    const int x = idx / N, c = idx % N;
    Uts[c * kMmaRows + mma_phys(x)] = (x < L) ? p.U[(size_t)x * N + c] : 0.0;
  }
  __syncthreads();

  const MmaLayout lay(Np);
  const int ldw = lay.ldw;
  unsigned char* ob = smem + p.ushared + (size_t)wid * p.owner_bytes;
  int* perm = reinterpret_cast<int*>(ob + lay.perm);
  int* pos = reinterpret_cast<int*>(ob + lay.pos);
  double* usel = reinterpret_cast<double*>(ob + lay.usel);
  double* Row = reinterpret_cast<double*>(ob + lay.row);
  double* Pinv = reinterpret_cast<double*>(ob + lay.pinv);
  double* Wf = reinterpret_cast<double*>(ob + lay.wf);
  double* Buf = reinterpret_cast<double*>(ob + lay.buf);
  for (int idx = lane; idx < Np * ldw; idx += G) Wf[idx] = 0.0;  // padding columns stay 0
  for (int idx = lane; idx < B * B; idx += G) Row[idx] = 0.0;

  // MMA-layout offsets (doubles) of this lane's A-fragment chunk in a U^T column, for the tile
  // pairs with a even / odd and round j: row x = 64a + 8g + 2j is chunk 32a + 4g + j, line
  // 4a + (g>>1), slot 4(g&1) + j; swizzled slot = (4(g&1) + j) ^ (4(a&1) + (g>>1)).
  const int g = lane >> 2, t4 = lane & 3;
  int aoff[2][4];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int j = 0; j < 4; ++j) aoff[h][j] = 2 * (8 * (g >> 1) + (((g & 1) ^ h) << 2) + (j ^ (g >> 1)));
  // transposition buffer: chunk (line l, slot s) holds the 16 bytes s ^ (l & 7) of lane l's row pair
  const int lsw = lane & 7;
  __syncwarp();

  for (int64_t id = (int64_t)blockIdx.x * nwarps + wid; id < p.M; id += (int64_t)gridDim.x * nwarps) {
    for (int j = lane; j < Np; j += G) {
      perm[j] = p.perm[id * Np + j] * kMmaRows;  // U^T column offset of m_j
      usel[j] = p.uniforms[id * 2 * (int64_t)Np + Np + j];
    }
    __syncwarp();
    uint32_t chosen = 0;
    int flag = 0;

    for (int k0 = 0; k0 < Np; k0 += B) {
      const int nb = min(B, Np - k0);
      double P[R][B];
      {
        // ---- a3 on the tensor path: acc = V[:, k0:k0+8] - V[:, 0:k0] W[0:k0, k0:k0+8]
        double acc[16][2][2];
        const int c0 = perm[min(k0 + 2 * t4, Np - 1)], c1 = perm[min(k0 + 2 * t4 + 1, Np - 1)];
#pragma unroll
        for (int pi = 0; pi < 16; ++pi) {
          const int j = pi >> 2, a = pi & 3;
          const int o = aoff[a & 1][j] + 64 * a;
          const double2 v0 = *reinterpret_cast<const double2*>(Uts + c0 + o);
          const double2 v1 = *reinterpret_cast<const double2*>(Uts + c1 + o);
          acc[pi][0][0] = v0.x;
          acc[pi][1][0] = v0.y;
          acc[pi][0][1] = v1.x;
          acc[pi][1][1] = v1.y;
        }
        const int kend = (p.dbg & 1) ? 0 : k0;
        for (int ks = 0; ks < kend; ks += 4) {
          const double* cb = Uts + perm[ks + t4];
          const double bf = -Wf[(ks + t4) * ldw + k0 + g];
#pragma unroll
          for (int pi = 0; pi < 16; ++pi) {
            const int j = pi >> 2, a = pi & 3;
            const double2 v = *reinterpret_cast<const double2*>(cb + aoff[a & 1][j] + 64 * a);
            dmma884(acc[pi][0][0], acc[pi][0][1], v.x, bf);
            dmma884(acc[pi][1][0], acc[pi][1][1], v.y, bf);
          }
        }
        // ---- MMA layout -> draw layout (rows 2j, 2j+1 of every lane per round)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          __syncwarp();
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int line = 8 * a + g;
              *reinterpret_cast<double2*>(Buf + 2 * (8 * line + ((4 * e + t4) ^ g))) =
                  make_double2(acc[4 * j + a][e][0], acc[4 * j + a][e][1]);
            }
          __syncwarp();
#pragma unroll
          for (int e = 0; e < 2; ++e)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const double2 v = *reinterpret_cast<const double2*>(Buf + 2 * (8 * lane + ((4 * e + q) ^ lsw)));
              P[2 * j + e][2 * q] = v.x;
              P[2 * j + e][2 * q + 1] = v.y;
            }
        }
      }
      if (nb < B) {  // ragged last block: columns past N' are zero
#pragma unroll
        for (int c = 1; c < B; ++c)
          if (c >= nb)
#pragma unroll
            for (int r = 0; r < R; ++r) P[r][c] = 0.0;
      }
      // rows drawn earlier get weight exactly 0 (the contraction leaves O(eps) residues)
#pragma unroll
      for (int r = 0; r < R; ++r) P[r][0] = ((chosen >> r) & 1u) ? 0.0 : P[r][0];

      // ---- a4/a5: nb sequential draws on the panel, one-column lookahead (as ffs_seg_kernel
      // OPT 135: kept partial sums, pivot row through shared memory, no warp vote)
      Draw dr;
      {
        double col0[R];
#pragma unroll
        for (int r = 0; r < R; ++r) col0[r] = P[r][0];
        dr = seg_draw<R, G, true>(col0, usel[k0], 0);
      }
      static_for<0, B>([&](auto rrc) {
        constexpr int rr = decltype(rrc)::value;
        if (rr < nb) {
          const int k = k0 + rr;
          int own, orow = 0;
          if (dr.ball != 0u) {
            own = __ffs(dr.ball) - 1;
          } else {
            // rare: u*T at/after the last partial sum, or T not finite/positive (reading Q5/Q8)
            double colr[R];
#pragma unroll
            for (int r = 0; r < R; ++r) colr[r] = P[r][rr];
            const int xf = seg_fallback<R, G>(colr, dr.T, chosen, L, lane, 0);
            own = xf / R;
            orow = xf % R;
          }
          if (!((dr.T > 0.0) && (dr.T <= 1.7976931348623157e308))) flag |= 1;
          if (p.trace != nullptr && id < p.S) {
            const double inv = dr.T > 0.0 ? 1.0 / dr.T : 0.0;
            double* tr = p.trace + (id * Np + k) * (int64_t)L;
#pragma unroll
            for (int r = 0; r < R; ++r)
              if (lane * R + r < L) tr[lane * R + r] = P[r][rr] * P[r][rr] * inv;
          }
          const double Tk = dr.T;
          const int rs = dr.ball != 0u ? dr.rsel : orow;
          // the owner lane stores row rs of its block (the pivot row) into Row
          const bool mine = (lane == own);
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
          const double pv = Row[rr * B + rr];
          if (pv * pv < 1e-12 * Tk) flag |= 2;
          const double ip = fast_rcp(pv);
          if (lane == 0) Pinv[rr] = ip;
          if constexpr (rr + 1 < B) {
            double sp[B];  // pivot row scaled by 1/pivot
#pragma unroll
            for (int c = rr + 1; c < B; c += 1) sp[c] = Row[rr * B + c] * ip;
            // column rr+1 first, then the next draw, then the remaining columns
#pragma unroll
            for (int r = 0; r < R; ++r)
              P[r][rr + 1] = ((chosen >> r) & 1u) ? 0.0 : fma(-P[r][rr], sp[rr + 1], P[r][rr + 1]);
            if (rr + 1 < nb) {
              double cn[R];
#pragma unroll
              for (int r = 0; r < R; ++r) cn[r] = P[r][rr + 1];
              dr = seg_draw<R, G, true>(cn, usel[k + 1], 0);
            }
#pragma unroll
            for (int c = rr + 2; c < B; ++c)
#pragma unroll
              for (int r = 0; r < R; ++r) P[r][c] = fma(-P[r][rr], sp[c], P[r][c]);
          }
        }
      });

      // ---- Gauss-Jordan update of W with the nb new rows (only if later columns remain)
      if (k0 + nb < Np && !(p.dbg & 4)) mma_gj(Uts, perm, pos, Row, Pinv, Wf, Buf, ldw, k0, Np, lane);
    }
    // ---- a6: positions and flags
    const unsigned fl = __reduce_or_sync(0xffffffffu, (unsigned)flag);
    for (int j = lane; j < Np; j += G) p.positions[id * Np + j] = pos[j];
    if (lane == 0 && p.flags != nullptr) p.flags[id] = fl & 3u;
    __syncwarp();
  }
}

}  // namespace ffsk
