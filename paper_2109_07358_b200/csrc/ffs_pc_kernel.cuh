// Warp-specialised FFS kernel for small real problems (L <= 32*R, N' <= kMaxNpWarp): the
// double-well headline workload.
//
// Same mathematics as ffs_warp_kernel.cuh / ffs_kernel.cuh (blocked left-looking randomized-pivot
// LU). The per-sample critical path alternates a throughput phase (panel
// contraction a3 + Gauss-Jordan update a2/a5, no dependency chain) with a latency phase (B
// sequential draws a4: scan, crossing search, pivot broadcast, rank-1 update). Instead of
// hoping that other warps happen to be in the other phase, every CTA pairs
//   * a CONSUMER warp, which only runs draws, and
//   * a PRODUCER warp, which only runs the Gauss-Jordan update and the next panel contraction,
// over TWO sample slots: while the consumer draws block b of slot 1, the producer finishes
// block b of slot 0 (Gauss-Jordan) and contracts its panel for block b+1, and vice versa.
// Panels travel through shared memory; the hand-off is an mbarrier pair per slot
// (full: panel ready, empty: block drawn).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ffs_warp_kernel.cuh"

namespace ffsk {

// per-sample shared-memory slice of the producer/consumer kernel
struct PcSlot {
  size_t perm, pos, usel, row, pinv, vnt, pbuf, wf, total;
  int ldw;
  __host__ __device__ PcSlot(int Np, int B, int R, bool wsmem) {
    ldw = (Np + B + 1) & ~1;
    size_t o = 0;
    perm = o; o = align16(o + sizeof(int) * Np);
    pos = o;  o = align16(o + sizeof(int) * Np);
    usel = o; o = align16(o + sizeof(double) * Np);
    row = o;  o = align16(o + sizeof(double) * B * B);
    pinv = o; o = align16(o + sizeof(double) * B);
    vnt = o;  o = align16(o + sizeof(double) * (size_t)Np * B);
    pbuf = o; o = align16(o + sizeof(double) * 32 * R * B);  // panel, [chunk][lane] of double2
    wf = o;   o = align16(o + (wsmem ? sizeof(double) * (size_t)Np * ldw : 0));  // W if in smem
    total = o;
  }
};

__host__ __device__ inline size_t pc_pair_bytes(int Np, int B, int R, bool wsmem) {
  return 2 * PcSlot(Np, B, R, wsmem).total + 64;  // two slots + 4 mbarriers (+ padding)
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared.b64 st, [%0];\n\t}" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}

template <int R, int B, int MAXT, bool WSMEM, bool TIMING = false>
__global__ void __launch_bounds__(MAXT, 1) ffs_pc_kernel(const WarpParams p) {
  long long tacc[5] = {0, 0, 0, 0, 0};
  long long tq = TIMING ? clock64() : 0;
#define PC_T0() do { if constexpr (TIMING) tq = clock64(); } while (0)
#define PC_T1(i) do { if constexpr (TIMING) { const long long t_ = clock64(); tacc[i] += t_ - tq; tq = t_; } } while (0)
  extern __shared__ __align__(16) unsigned char smem[];
  using Sw = Swz<double, R>;
  constexpr int G = 32;
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int npairs = blockDim.x >> 6;
  // consumers get the HIGHER warp ids: the warp arbiter prefers high ids, so the latency-critical
  // draw chain issues first and the producer's contraction fills the remaining slots
  const bool consumer = wid >= npairs;
  const int pair = consumer ? wid - npairs : wid;
  const int L = p.L, N = p.N, Np = p.Np;
  const int stride = p.ut_stride;

  // ---- U^T into shared memory (swizzled 16-byte chunks; rows >= L zero)
  double* Uts = reinterpret_cast<double*>(smem);
  for (int idx = threadIdx.x; idx < N * p.Lp; idx += blockDim.x) {
    const int x = idx / N, c = idx % N;
    Uts[(size_t)c * stride + Sw::phys(x)] = (x < L) ? p.U[(size_t)x * N + c] : 0.0;
  }
  const PcSlot lay(Np, B, R, WSMEM);
  const int ldw = lay.ldw;
  unsigned char* pb = smem + p.ushared + (size_t)pair * p.owner_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(pb + 2 * lay.total);  // full[0..1], empty[0..1]
  if (consumer && lane == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(bars + i, 1);
  }
  __syncthreads();

  auto slot = [&](int s) { return pb + (size_t)s * lay.total; };
  const int nblk = (Np + B - 1) / B;
  const int64_t gpair = (int64_t)blockIdx.x * npairs + pair;
  const int64_t tpairs = (int64_t)gridDim.x * npairs;
  const int64_t ngroups = (p.M + 1) / 2;

  if (!consumer) {
    // ============================ PRODUCER ============================
    const int sw = Sw::sw(lane);
    const double* Ucol0 = Uts + lane * R;
    int qoff[R / 2];
#pragma unroll
    for (int q = 0; q < R / 2; ++q) qoff[q] = (q ^ sw) << 1;
    // W = A^{-1} V[X, later cols] per slot, in global memory (L2-resident: 2 x N' x ldw doubles)
    double* Wbase = WSMEM ? nullptr : p.wfull + (size_t)gpair * 2 * Np * ldw;
    for (int s = 0; s < 2; ++s) {
      double* Wf = WSMEM ? reinterpret_cast<double*>(slot(s) + lay.wf) : Wbase + (size_t)s * Np * ldw;
      for (int idx = lane; idx < Np * ldw; idx += 32) Wf[idx] = 0.0;  // padding cols stay 0
    }
    for (int s = 0; s < 2; ++s) {
      double* Row = reinterpret_cast<double*>(slot(s) + lay.row);
      for (int idx = lane; idx < B * B; idx += 32) Row[idx] = 0.0;
    }
    __syncwarp();
    unsigned pe[2] = {0u, 0u};  // completed waits on empty[s]
    for (int64_t g = gpair; g < ngroups; g += tpairs) {
      bool live[2];
#pragma unroll
      for (int s = 0; s < 2; ++s) live[s] = g * 2 + s < p.M;
      for (int b = 0; b < nblk; ++b) {
        const int k0 = b * B;
        const int nb = min(B, Np - k0);
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          if (!live[s]) continue;
          const int64_t id = g * 2 + s;
          int* perm = reinterpret_cast<int*>(slot(s) + lay.perm);
          double* Wf = WSMEM ? reinterpret_cast<double*>(slot(s) + lay.wf) : Wbase + (size_t)s * Np * ldw;
          if (b == 0) {
            if (g != gpair) {  // previous sample of this slot fully drawn and written out
              PC_T0();
              mbar_wait(bars + 2 + s, pe[s] & 1u);
              ++pe[s];
              PC_T1(0);
            }
            double* usel = reinterpret_cast<double*>(slot(s) + lay.usel);
            for (int j = lane; j < Np; j += 32) {
              perm[j] = p.perm[id * Np + j];
              usel[j] = p.uniforms[id * 2 * (int64_t)Np + Np + j];
            }
            __syncwarp();
          } else {
            // ---- wait for the draws of block b-1, then Gauss-Jordan update of W with its rows
            PC_T0();
            mbar_wait(bars + 2 + s, pe[s] & 1u);
            ++pe[s];
            PC_T1(0);
            const int kp = k0 - B;  // start of block b-1 (full width B)
            const int* pos = reinterpret_cast<const int*>(slot(s) + lay.pos);
            const double* Row = reinterpret_cast<const double*>(slot(s) + lay.row);
            const double* Pinv = reinterpret_cast<const double*>(slot(s) + lay.pinv);
            double* VnT = reinterpret_cast<double*>(slot(s) + lay.vnt);
            for (int idx = lane; idx < Np * B; idx += 32) {
              const int ii = idx / B, tt = idx % B;
              VnT[idx] = Uts[perm[ii] * stride + Sw::phys(pos[kp + tt])];
            }
            __syncwarp();
            double ipv[B];
#pragma unroll
            for (int t2 = 0; t2 < B; ++t2) ipv[t2] = Pinv[t2];
            for (int j = k0 + lane; j < Np; j += 32) {
              double z[B];
#pragma unroll
              for (int tt = 0; tt < B; ++tt) z[tt] = VnT[j * B + tt];
              int ii = 0;
              for (; ii + 4 <= kp; ii += 4) {  // 4 independent W loads in flight
                double w4[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) w4[u] = Wf[(ii + u) * ldw + j];
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                  for (int tt = 0; tt < B; tt += 2) {
                    const double2 v = *reinterpret_cast<const double2*>(VnT + (ii + u) * B + tt);
                    z[tt] = fma(-v.x, w4[u], z[tt]);
                    z[tt + 1] = fma(-v.y, w4[u], z[tt + 1]);
                  }
              }
              for (; ii < kp; ++ii) {
                const double wij = Wf[ii * ldw + j];
#pragma unroll
                for (int tt = 0; tt < B; tt += 2) {
                  const double2 v = *reinterpret_cast<const double2*>(VnT + ii * B + tt);
                  z[tt] = fma(-v.x, wij, z[tt]);
                  z[tt + 1] = fma(-v.y, wij, z[tt + 1]);
                }
              }
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
              ii = 0;
              for (; ii + 4 <= kp; ii += 4) {
                double a4[4], wb4[4][B];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  a4[u] = Wf[(ii + u) * ldw + j];
#pragma unroll
                  for (int tt = 0; tt < B; tt += 2) {
                    const double2 wbv = *reinterpret_cast<const double2*>(Wf + (ii + u) * ldw + kp + tt);
                    wb4[u][tt] = wbv.x;
                    wb4[u][tt + 1] = wbv.y;
                  }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
#pragma unroll
                  for (int tt = 0; tt < B; ++tt) a4[u] = fma(-wb4[u][tt], z[tt], a4[u]);
                  Wf[(ii + u) * ldw + j] = a4[u];
                }
              }
              for (; ii < kp; ++ii) {
                double a = Wf[ii * ldw + j];
#pragma unroll
                for (int tt = 0; tt < B; tt += 2) {
                  const double2 wbv = *reinterpret_cast<const double2*>(Wf + ii * ldw + kp + tt);
                  a = fma(-wbv.x, z[tt], a);
                  a = fma(-wbv.y, z[tt + 1], a);
                }
                Wf[ii * ldw + j] = a;
              }
#pragma unroll
              for (int tt = 0; tt < B; ++tt) Wf[(kp + tt) * ldw + j] = z[tt];
            }
            __syncwarp();
          }
          PC_T1(1);
          // ---- a3 panel of block b: P = V[:, k0:k0+B] - V[:, 0:k0] W[0:k0, k0:k0+B]
          double P[R][B];
#pragma unroll
          for (int c = 0; c < B; ++c) {
            const double* cb = Ucol0 + perm[min(k0 + c, Np - 1)] * stride;
#pragma unroll
            for (int q = 0; q < R / 2; ++q) {
              const double2 d = *reinterpret_cast<const double2*>(cb + qoff[q]);
              P[2 * q][c] = (c < nb) ? d.x : 0.0;
              P[2 * q + 1][c] = (c < nb) ? d.y : 0.0;
            }
          }
          {
            const double* wrow = Wf + k0;
#pragma unroll 4
            for (int ii = 0; ii < k0; ++ii, wrow += ldw) {
              const double* cb = Ucol0 + perm[ii] * stride;
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
          // hand the panel to the consumer: [chunk j = (row pair, column)][lane] of double2
          double2* pbuf = reinterpret_cast<double2*>(slot(s) + lay.pbuf);
#pragma unroll
          for (int q = 0; q < R / 2; ++q)
#pragma unroll
            for (int c = 0; c < B; ++c) pbuf[(q * B + c) * 32 + lane] = make_double2(P[2 * q][c], P[2 * q + 1][c]);
          __syncwarp();
          if (lane == 0) mbar_arrive(bars + s);
          PC_T1(2);
        }
      }
    }
    if constexpr (TIMING) {
      if (lane == 0 && p.timing != nullptr)
        for (int q = 0; q < 3; ++q) atomicAdd(p.timing + q, (unsigned long long)tacc[q]);
    }
    return;
  }

  // ============================ CONSUMER ============================
  unsigned cf[2] = {0u, 0u};  // completed waits on full[s]
  for (int64_t g = gpair; g < ngroups; g += tpairs) {
    bool live[2];
    uint32_t chosen[2] = {0u, 0u};
    int flag[2] = {0, 0};
#pragma unroll
    for (int s = 0; s < 2; ++s) live[s] = g * 2 + s < p.M;
    for (int b = 0; b < nblk; ++b) {
      const int k0 = b * B;
      const int nb = min(B, Np - k0);
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        if (!live[s]) continue;
        const int64_t id = g * 2 + s;
        int* pos = reinterpret_cast<int*>(slot(s) + lay.pos);
        const double* usel = reinterpret_cast<const double*>(slot(s) + lay.usel);
        double* Row = reinterpret_cast<double*>(slot(s) + lay.row);
        double* Pinv = reinterpret_cast<double*>(slot(s) + lay.pinv);
        PC_T0();
        mbar_wait(bars + s, cf[s] & 1u);
        ++cf[s];
        PC_T1(3);
        double P[R][B];
        {
          const double2* pbuf = reinterpret_cast<const double2*>(slot(s) + lay.pbuf);
#pragma unroll
          for (int q = 0; q < R / 2; ++q)
#pragma unroll
            for (int c = 0; c < B; ++c) {
              const double2 d = pbuf[(q * B + c) * 32 + lane];
              P[2 * q][c] = d.x;
              P[2 * q + 1][c] = d.y;
            }
        }
        uint32_t ch = chosen[s];
        int fl = flag[s];
        // rows drawn earlier: weight exactly 0 in the column of the next draw
#pragma unroll
        for (int r = 0; r < R; ++r) P[r][0] = ((ch >> r) & 1u) ? 0.0 : P[r][0];
        Draw dr;
        {
          double col0[R];
#pragma unroll
          for (int r = 0; r < R; ++r) col0[r] = P[r][0];
          dr = seg_draw<R, G>(col0, usel[k0], 0);
        }
        static_for<0, B>([&](auto rrc) {
          constexpr int rr = decltype(rrc)::value;
          if (rr < nb) {
            const int k = k0 + rr;
            int own, orow;
            if (dr.ball != 0u) {
              own = __ffs(dr.ball) - 1;
              orow = __shfl_sync(0xffffffffu, dr.rsel, own);
            } else {  // rare: u*T at/after the last partial sum, or T not finite/positive
              double colr[R];
#pragma unroll
              for (int r = 0; r < R; ++r) colr[r] = P[r][rr];
              const int xf = seg_fallback<R, G>(colr, dr.T, ch, L, lane, 0);
              own = xf / R;
              orow = xf % R;
            }
            if (!((dr.T > 0.0) && isfinite(dr.T))) fl |= 1;
            if (p.trace != nullptr && id < p.S) {
              const double inv = dr.T > 0.0 ? 1.0 / dr.T : 0.0;
              double* tr = p.trace + (id * Np + k) * (int64_t)L;
#pragma unroll
              for (int r = 0; r < R; ++r)
                if (lane * R + r < L) tr[lane * R + r] = P[r][rr] * P[r][rr] * inv;
            }
            // pivot row: every lane selects row rs of its block (select tree), owner broadcasts
            const int rs = dr.ball != 0u ? dr.rsel : orow;
            double prow[B];
#pragma unroll
            for (int c = 0; c < B; ++c) {
              double t[R];
#pragma unroll
              for (int r = 0; r < R; ++r) t[r] = P[r][c];
#pragma unroll
              for (int w = 1; w < R; w <<= 1)
#pragma unroll
                for (int i = 0; i < R; i += 2 * w) t[i] = (rs & w) ? t[i + w] : t[i];
              prow[c] = __shfl_sync(0xffffffffu, t[0], own);
            }
            ch |= (lane == own) ? (1u << orow) : 0u;
            if (prow[rr] * prow[rr] < 1e-12 * dr.T) fl |= 2;
            const double ip = fast_rcp(prow[rr]);
            if (lane == 0) {
              pos[k] = own * R + orow;
              Pinv[rr] = ip;
#pragma unroll
              for (int c = 0; c < B; c += 2)
                *reinterpret_cast<double2*>(Row + rr * B + c) = make_double2(prow[c], prow[c + 1]);
            }
            if constexpr (rr + 1 < B) {
              double sp[B];
#pragma unroll
              for (int c = rr + 1; c < B; ++c) sp[c] = prow[c] * ip;
#pragma unroll
              for (int r = 0; r < R; ++r)
                P[r][rr + 1] = ((ch >> r) & 1u) ? 0.0 : fma(-P[r][rr], sp[rr + 1], P[r][rr + 1]);
              if (rr + 1 < nb) {
                double cn[R];
#pragma unroll
                for (int r = 0; r < R; ++r) cn[r] = P[r][rr + 1];
                dr = seg_draw<R, G>(cn, usel[k + 1], 0);
              }
#pragma unroll
              for (int c = rr + 2; c < B; ++c)
#pragma unroll
                for (int r = 0; r < R; ++r) P[r][c] = fma(-P[r][rr], sp[c], P[r][c]);
            }
          }
        });
        chosen[s] = ch;
        flag[s] = fl;
        if (b == nblk - 1) {  // sample done: positions and flags out
          __syncwarp();
          const int f = __reduce_or_sync(0xffffffffu, fl);
          for (int j = lane; j < Np; j += 32) p.positions[id * Np + j] = pos[j];
          if (lane == 0 && p.flags != nullptr) p.flags[id] = f;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(bars + 2 + s);
        PC_T1(4);
      }
    }
  }
  if constexpr (TIMING) {
    if (lane == 0 && p.timing != nullptr)
      for (int q = 3; q < 5; ++q) atomicAdd(p.timing + q, (unsigned long long)tacc[q]);
  }
#undef PC_T0
#undef PC_T1
}

}  // namespace ffsk
