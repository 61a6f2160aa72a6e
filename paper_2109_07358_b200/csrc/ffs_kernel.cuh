// FFS sampling kernel for sm_100a: batched, per-sample randomized-pivot LU in the
// blocked left-looking form, one persistent "owner" (a warp, or a whole CTA) per sample.
//
// What is computed (Eq. 3; Supp S1 PAPER.md:248-256) for one sample, with
// V = U[:, m] the permuted columns (never materialised), X_k = (x_1..x_k) the chosen rows and
// A_k = V[X_k, 0:k]:
//   the step-k weight of site x is |s_k(x)|^2 with s_k(x) = V[x,k] - V[x,0:k] A_k^{-1} V[X_k,k]
//   (= u_x^T h' with the un-normalised normal vector h' = (-A^{-1}V[X,k]; 1) of Eq. 3; the
//   normalisation |h'|^2 cancels in the inverse-CDF draw).
// s_k is the k-th column of the Schur complement of V after eliminating the chosen rows, i.e.
// FFS is an LU factorisation of V whose pivot row in column k is DRAWN with probability
// ∝ |Schur entry|^2. The kernel computes it in blocks of B columns:
//   (1) panel:   P = V[:, k0:k0+B] - V[:, 0:k0] Wb,  Wb = A_{k0}^{-1} V[X_{k0}, k0:k0+B]
//                (L x k0 x B contraction per sample; V gathered from U by the sample's m)
//   (2) B sequential steps on the register-resident panel: weights |P[:,r]|^2 (chosen rows 0),
//       group scan + inverse-CDF select, broadcast of the pivot row, rank-1 update of the
//       remaining panel columns (right-looking).
//   (3) Gauss-Jordan update of W = A^{-1} V[X, k0+B:N'] (all later columns) with the B new rows,
//       using the LU of the B x B Schur block that step (2) produced.
// This replaces the paper's eager full-N elimination (S1) + per-step back-substitution; the
// executed flop count is L N'^2 + O(N'^3) per sample.
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "ffs_scalar.cuh"

namespace ffsk {

struct Params {
  const double* U;         // row-major [L][N] scalars (complex interleaved)
  const double* Ut;        // transposed, zero-padded [N][Lp] scalars (global path)
  int L, N, Np, Lp;        // Lp = rows covered by one owner (G*R)
  int ut_stride;           // smem column stride in scalars (shared-U path)
  int64_t M;
  const double* uniforms;  // [M][2Np]
  int32_t* positions;      // [M][Np]
  int32_t* flags;          // [M] or null
  double* wfull;           // per owner [Np][Np] scalars
  int64_t S0, S;           // debug trace of samples S0 .. S0+S-1
  double* trace;           // [S][Np][L] or null
  size_t owner_smem;       // bytes of per-owner shared memory
  size_t ushared_smem;     // bytes of the shared U^T copy (shared-U path)
  // ragged mode (L-ensemble front end, ffs_lens.cu): sample i runs nps[i] <= Np steps on the
  // columns cols[i][0 .. nps[i]) (its kept eigenvectors, already permuted); null otherwise
  const int32_t* cols;     // [M][N]
  const int32_t* nps;      // [M]
  int ustride;             // uniform row stride: 2 Np (ffs_sample), 3 N (L-ensemble)
  int usel;                // offset of the selection uniforms within a row: Np, or 2 N
};

__host__ __device__ inline size_t align16(size_t v) { return (v + 15) & ~size_t(15); }

template <typename T, int B>
struct OwnerLayout {
  size_t perm, pos, row, pinv, wb, vnew, red, redi, total;
  __host__ __device__ OwnerLayout(int N, int Np) {
    size_t o = 0;
    perm = o; o = align16(o + sizeof(int) * N);
    pos = o;  o = align16(o + sizeof(int) * Np);
    row = o;  o = align16(o + sizeof(T) * B * B);
    pinv = o; o = align16(o + sizeof(T) * B);
    wb = o;   o = align16(o + sizeof(T) * (size_t)Np * B);
    vnew = o; o = align16(o + sizeof(T) * (size_t)Np * B);
    red = o;  o = align16(o + sizeof(double) * 32);
    redi = o; o = align16(o + sizeof(int) * 96);
    total = o;
  }
};

// ---- swizzled shared-memory U^T: thread t of an owner holds rows t*R .. t*R+R-1; those rows
// are stored as 16-byte chunks XOR-swizzled by the thread index so that the per-thread
// vector loads of one column are bank-conflict free (8 lanes per 128-byte phase).
template <typename T, int R>
struct Swz {
  static constexpr int kChunkScalars = sizeof(T) == 8 ? 2 : 1;           // scalars per 16 B
  static constexpr int C = (R >= kChunkScalars) ? R / kChunkScalars : 0;  // chunks per thread
  __host__ __device__ static int lanes_per_row() { return C >= 8 ? 1 : (C > 0 ? 8 / C : 8); }
  __host__ __device__ static int sw(int t) {
    if (C <= 1) return 0;
    int m = C < 8 ? C : 8;
    return (t / lanes_per_row()) & (m - 1);
  }
  // physical index (in scalars, within a column) of logical row x
  __host__ __device__ static int phys(int x) {
    if (C == 0) return x;
    int t = x / R, w = x % R;
    int q = w / kChunkScalars, e = w % kChunkScalars;
    return t * R + (q ^ sw(t)) * kChunkScalars + e;
  }
};

// store one 16-byte chunk (2 real or 1 complex scalar) into a register array, constant index q
template <typename T, int R>
__device__ __forceinline__ void set_chunk(T (&v)[R], int q, double2 d) {
  if constexpr (sizeof(T) == 8) {
    v[2 * q] = d.x;
    v[2 * q + 1] = d.y;
  } else {
    v[q].re = d.x;
    v[q].im = d.y;
  }
}

template <int I, int N, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (I < N) {
    f(std::integral_constant<int, I>{});
    static_for<I + 1, N>(f);
  }
}

template <typename T, int R, bool USMEM>
__device__ __forceinline__ void load_col(const Params& p, const T* __restrict__ Uts, int col, int t,
                                         T (&v)[R]) {
  if constexpr (USMEM) {
    const T* base = Uts + (size_t)col * p.ut_stride + t * R;
    using S = Swz<T, R>;
    if constexpr (S::C == 0) {
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = base[r];
    } else {
      const int s = S::sw(t);
#pragma unroll
      for (int q = 0; q < S::C; ++q) {
        const double2 d = *reinterpret_cast<const double2*>(base + (q ^ s) * S::kChunkScalars);
        set_chunk<T, R>(v, q, d);
      }
    }
  } else {
    const T* base = reinterpret_cast<const T*>(p.Ut) + (size_t)col * p.Lp + t * R;
    if constexpr (sizeof(T) == 8 && (R % 4) == 0) {  // 32-byte loads (Lp is a multiple of R)
#pragma unroll
      for (int q = 0; q < R / 4; ++q)
        asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
            : "=d"(v[4 * q]), "=d"(v[4 * q + 1]), "=d"(v[4 * q + 2]), "=d"(v[4 * q + 3])
            : "l"(base + 4 * q));
    } else if constexpr (sizeof(T) == 8 && (R % 2) == 0) {
#pragma unroll
      for (int q = 0; q < R / 2; ++q) {
        const double2 d = __ldg(reinterpret_cast<const double2*>(base) + q);
        set_chunk<T, R>(v, q, d);
      }
    } else if constexpr (sizeof(T) == 16) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double2 d = __ldg(reinterpret_cast<const double2*>(base) + r);
        set_chunk<T, R>(v, r, d);
      }
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = reinterpret_cast<const T*>(&p.Ut[0])[(size_t)col * p.Lp + t * R + r];
    }
  }
}

template <bool WARP>
__device__ __forceinline__ void gsync() {
  if constexpr (WARP) __syncwarp();
  else __syncthreads();
}

__device__ __forceinline__ double warp_incl_scan(double v, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    double y = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += y;
  }
  return v;
}

// Inverse-CDF selection over the owner's L weights (reading Q5 in DESIGN.md):
//   T = sum w; x_k = min{x : C(x) > u*T, w(x) > 0}; fallback: the largest x with w(x) > 0;
//   if T is not finite and positive: the smallest unchosen site (the caller flags bit0).
// Thread t owns rows t*R..t*R+R-1 (index order = scan order). Returns x_k (owner-uniform).
template <bool WARP, int R>
__device__ __forceinline__ int select_site(const double (&w)[R], double u, int t, int L, uint32_t chosen,
                                           double* red, int* redi, double& T_out) {
  const int lane = t & 31;
  const int warp = t >> 5;
  double c[R];
  double acc = 0.0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    acc += w[r];
    c[r] = acc;
  }
  const double incl = warp_incl_scan(acc, lane);
  double excl = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 0) excl = 0.0;
  double T;
  int nw = 1;
  if constexpr (WARP) {
    T = __shfl_sync(0xffffffffu, incl, 31);
  } else {
    nw = blockDim.x >> 5;
    if (lane == 31) red[warp] = incl;
    __syncthreads();
    const double wt = lane < nw ? red[lane] : 0.0;
    const double ws = warp_incl_scan(wt, lane);
    const double woff = __shfl_sync(0xffffffffu, ws, warp > 0 ? warp - 1 : 0);
    T = __shfl_sync(0xffffffffu, ws, 31);
    if (warp > 0) excl += woff;
  }
  const bool ok = (T > 0.0) && isfinite(T);
  const double thr = u * T;
  int rfirst = R, rlast = -1, rfree = R;
#pragma unroll
  for (int r = R - 1; r >= 0; --r) {
    if (w[r] > 0.0 && excl + c[r] > thr) rfirst = r;
    if (t * R + r < L && !((chosen >> r) & 1u)) rfree = r;
  }
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (w[r] > 0.0) rlast = r;
  constexpr int kNone = 0x7fffffff;
  int cf = kNone, cl = -1, cu = kNone;
  {
    const unsigned b1 = __ballot_sync(0xffffffffu, rfirst < R);
    if (b1) {
      const int ln = __ffs(b1) - 1;
      cf = ((warp << 5) + ln) * R + __shfl_sync(0xffffffffu, rfirst, ln);
    }
    const unsigned b2 = __ballot_sync(0xffffffffu, rlast >= 0);
    if (b2) {
      const int ln = 31 - __clz(b2);
      cl = ((warp << 5) + ln) * R + __shfl_sync(0xffffffffu, rlast, ln);
    }
    const unsigned b3 = __ballot_sync(0xffffffffu, rfree < R);
    if (b3) {
      const int ln = __ffs(b3) - 1;
      cu = ((warp << 5) + ln) * R + __shfl_sync(0xffffffffu, rfree, ln);
    }
  }
  if constexpr (!WARP) {
    if (lane == 0) {
      redi[warp] = cf;
      redi[32 + warp] = cl;
      redi[64 + warp] = cu;
    }
    __syncthreads();
    cf = __reduce_min_sync(0xffffffffu, lane < nw ? redi[lane] : kNone);
    cl = __reduce_max_sync(0xffffffffu, lane < nw ? redi[32 + lane] : -1);
    cu = __reduce_min_sync(0xffffffffu, lane < nw ? redi[64 + lane] : kNone);
  }
  T_out = T;
  if (!ok) return cu;
  return cf != kNone ? cf : cl;
}

template <typename T, bool WARP, int R, int B, bool USMEM, int MAXT>
__global__ void __launch_bounds__(MAXT)
ffs_sample_kernel(const Params p) {
  extern __shared__ __align__(16) unsigned char smem[];
  using S = Sc<T>;
  const int G = WARP ? 32 : blockDim.x;
  const int owners_per_cta = WARP ? (blockDim.x >> 5) : 1;
  const int t = WARP ? (threadIdx.x & 31) : threadIdx.x;
  const int oidx = WARP ? (threadIdx.x >> 5) : 0;
  const int L = p.L, N = p.N, Np = p.Np;

  const T* Uts = reinterpret_cast<const T*>(smem);
  if constexpr (USMEM) {
    // cooperative, swizzled transpose of U [L][N] -> smem U^T [N][stride] (rows >= L are zero)
    T* dst = reinterpret_cast<T*>(smem);
    const T* src = reinterpret_cast<const T*>(p.U);
    const int total = N * p.Lp;
    for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
      const int x = idx / N, c = idx % N;
      T v = (x < L) ? src[(size_t)x * N + c] : S::zero();
      dst[(size_t)c * p.ut_stride + Swz<T, R>::phys(x)] = v;
    }
    __syncthreads();
  }
  const OwnerLayout<T, B> lay(N, Np);
  unsigned char* ob = smem + p.ushared_smem + (size_t)oidx * p.owner_smem;
  int* perm = reinterpret_cast<int*>(ob + lay.perm);
  int* pos = reinterpret_cast<int*>(ob + lay.pos);
  T* Row = reinterpret_cast<T*>(ob + lay.row);
  T* Pinv = reinterpret_cast<T*>(ob + lay.pinv);
  T* Wb = reinterpret_cast<T*>(ob + lay.wb);
  T* Vnew = reinterpret_cast<T*>(ob + lay.vnew);
  double* red = reinterpret_cast<double*>(ob + lay.red);
  int* redi = reinterpret_cast<int*>(ob + lay.redi);

  const int64_t gid = (int64_t)blockIdx.x * owners_per_cta + oidx;
  const int64_t num_owners = (int64_t)gridDim.x * owners_per_cta;
  T* Wf = reinterpret_cast<T*>(p.wfull) + gid * (int64_t)Np * Np;
  const T* Ug = reinterpret_cast<const T*>(p.U);

  for (int64_t i = gid; i < p.M; i += num_owners) {
    const double* urow = p.uniforms + i * (int64_t)p.ustride;
    const double* usel = urow + p.usel;
    const int Npi = p.nps ? p.nps[i] : Np;  // steps of this sample (ragged mode: its N_i)
    if (p.cols) {
      // ragged mode: the permuted kept columns come precomputed
      for (int j = t; j < Npi; j += G) {
        FFS_CHECK(p.cols[i * N + j] >= 0 && p.cols[i * N + j] < N);
        perm[j] = p.cols[i * N + j];
      }
    } else {
      // ---- a1: permutation (reading Q6), forward partial Fisher-Yates
      for (int j = t; j < N; j += G) perm[j] = j;
      gsync<WARP>();
      if (t == 0) {
        for (int j = 0; j < Np; ++j) {
          const int n = N - j;
          int r = (int)floor(urow[j] * (double)n);
          r = (r > n - 1 ? n - 1 : r) + j;
          const int a = perm[j];
          perm[j] = perm[r];
          perm[r] = a;
        }
      }
    }
    gsync<WARP>();
    uint32_t chosen = 0;
    int flag = 0;

    for (int k0 = 0; k0 < Npi; k0 += B) {
      const int nb = min(B, Npi - k0);
      // ---- stage Wb = W[0:k0, k0:k0+nb] (A^{-1} V[X, block cols])
      for (int idx = t; idx < k0 * B; idx += G) {
        const int ii = idx / B, c = idx % B;
        Wb[idx] = c < nb ? Wf[(size_t)ii * Npi + k0 + c] : S::zero();
      }
      gsync<WARP>();
      // ---- a3: panel P = V[:, k0:k0+B] - V[:, 0:k0] Wb   (registers: R rows x B cols)
      T P[R][B];
#pragma unroll
      for (int c = 0; c < B; ++c) {
        T v[R];
        if (c < nb) {
          load_col<T, R, USMEM>(p, Uts, perm[k0 + c], t, v);
        } else {
#pragma unroll
          for (int r = 0; r < R; ++r) v[r] = S::zero();
        }
#pragma unroll
        for (int r = 0; r < R; ++r) P[r][c] = v[r];
      }
#pragma unroll 4
      for (int ii = 0; ii < k0; ++ii) {
        T v[R];
        load_col<T, R, USMEM>(p, Uts, perm[ii], t, v);
        T wb[B];
#pragma unroll
        for (int c = 0; c < B; ++c) wb[c] = Wb[ii * B + c];
#pragma unroll
        for (int c = 0; c < B; ++c)
#pragma unroll
          for (int r = 0; r < R; ++r) P[r][c] = S::fms(v[r], wb[c], P[r][c]);
      }
      // ---- a4/a5: B sequential steps on the panel
      static_for<0, B>([&](auto rrc) {
        constexpr int rr = decltype(rrc)::value;
        if (rr < nb) {
          const int k = k0 + rr;
          double w[R];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int x = t * R + r;
            w[r] = (x < L && !((chosen >> r) & 1u)) ? S::abs2(P[r][rr]) : 0.0;
          }
          double Ttot;
          const int xk = select_site<WARP, R>(w, usel[k], t, L, chosen, red, redi, Ttot);
          if (!((Ttot > 0.0) && isfinite(Ttot))) flag |= 1;
          const int own = xk / R, orow = xk % R;
          if (t == own) {
            // pivot row (and, in columns < rr, the Schur values that become L-multipliers)
#pragma unroll
            for (int r = 0; r < R; ++r)
              if (r == orow) {
#pragma unroll
                for (int c = 0; c < B; ++c) Row[rr * B + c] = P[r][c];
                if (Ttot > 0.0 && w[r] / Ttot < 1e-12) flag |= 2;
              }
            pos[k] = xk;
          }
          if (p.trace != nullptr && (uint64_t)(i - p.S0) < (uint64_t)p.S) {
            double inv = Ttot > 0.0 ? 1.0 / Ttot : 0.0;
            double* tr = p.trace + ((i - p.S0) * Np + k) * (int64_t)L;
#pragma unroll
            for (int r = 0; r < R; ++r)
              if (t * R + r < L) tr[t * R + r] = w[r] * inv;
          }
          gsync<WARP>();
          const T piv = Row[rr * B + rr];
          const T ip = S::recip(piv);
          if (t == 0) Pinv[rr] = ip;
          T lmul[R];
#pragma unroll
          for (int r = 0; r < R; ++r) lmul[r] = S::mul(P[r][rr], ip);
#pragma unroll
          for (int c = rr + 1; c < B; ++c) {
            const T pc = Row[rr * B + c];
#pragma unroll
            for (int r = 0; r < R; ++r) P[r][c] = S::fms(lmul[r], pc, P[r][c]);
          }
          if (t == own) chosen |= 1u << orow;
        }
      });
      // ---- Gauss-Jordan update of W with the nb new rows (only if later columns remain)
      if (k0 + nb < Npi) {
        gsync<WARP>();
        for (int idx = t; idx < nb * Npi; idx += G) {
          const int tt = idx / Npi, j = idx % Npi;
          Vnew[idx] = Ug[(size_t)pos[k0 + tt] * N + perm[j]];
        }
        gsync<WARP>();
        for (int j = k0 + nb + t; j < Npi; j += G) {
          T z[B];
#pragma unroll
          for (int tt = 0; tt < B; ++tt) z[tt] = tt < nb ? Vnew[tt * Npi + j] : S::zero();
          // R_new = V[X_new, j] - V[X_new, 0:k0] W[0:k0, j]; 8 independent W loads in flight
          int ii = 0;
          for (; ii + 8 <= k0; ii += 8) {
            T w8[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) w8[u] = Wf[(size_t)(ii + u) * Npi + j];
#pragma unroll
            for (int u = 0; u < 8; ++u)
#pragma unroll
              for (int tt = 0; tt < B; ++tt)
                if (tt < nb) z[tt] = S::fms(Vnew[tt * Npi + ii + u], w8[u], z[tt]);
          }
          for (; ii < k0; ++ii) {
            const T wij = Wf[(size_t)ii * Npi + j];
#pragma unroll
            for (int tt = 0; tt < B; ++tt)
              if (tt < nb) z[tt] = S::fms(Vnew[tt * Npi + ii], wij, z[tt]);
          }
          // forward substitution with the unit-lower factor L[tt][s] = Row[tt][s] * Pinv[s]
#pragma unroll
          for (int tt = 1; tt < B; ++tt)
            if (tt < nb) {
#pragma unroll
              for (int s = 0; s < tt; ++s) z[tt] = S::fms(S::mul(Row[tt * B + s], Pinv[s]), z[s], z[tt]);
            }
          // back substitution with the upper factor U[tt][s] = Row[tt][s] (s >= tt)
#pragma unroll
          for (int tt = B - 1; tt >= 0; --tt)
            if (tt < nb) {
#pragma unroll
              for (int s = tt + 1; s < B; ++s)
                if (s < nb) z[tt] = S::fms(Row[tt * B + s], z[s], z[tt]);
              z[tt] = S::mul(z[tt], Pinv[tt]);
            }
#pragma unroll
          for (int tt = 0; tt < B; ++tt)
            if (tt < nb) Wf[(size_t)(k0 + tt) * Npi + j] = z[tt];
          // W[0:k0, j] -= Wb Z[:, j]; 8 rows per batch (independent loads, then stores)
          ii = 0;
          for (; ii + 8 <= k0; ii += 8) {
            T a8[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) a8[u] = Wf[(size_t)(ii + u) * Npi + j];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
#pragma unroll
              for (int tt = 0; tt < B; ++tt)
                if (tt < nb) a8[u] = S::fms(Wb[(ii + u) * B + tt], z[tt], a8[u]);
              Wf[(size_t)(ii + u) * Npi + j] = a8[u];
            }
          }
          for (; ii < k0; ++ii) {
            T a = Wf[(size_t)ii * Npi + j];
#pragma unroll
            for (int tt = 0; tt < B; ++tt)
              if (tt < nb) a = S::fms(Wb[ii * B + tt], z[tt], a);
            Wf[(size_t)ii * Npi + j] = a;
          }
        }
      }
      gsync<WARP>();
    }
    // ---- a6: positions (sampling order) and flags
    for (int j = t; j < Np; j += G) {
      FFS_CHECK(j >= Npi || (pos[j] >= 0 && pos[j] < L));
      p.positions[i * Np + j] = j < Npi ? pos[j] : -1;
    }
    if constexpr (WARP) {
      flag = __reduce_or_sync(0xffffffffu, flag);
    } else {
      flag = (__syncthreads_or(flag & 1) ? 1 : 0) | (__syncthreads_or(flag & 2) ? 2 : 0);
    }
    if (t == 0 && p.flags != nullptr) p.flags[i] = flag;
    gsync<WARP>();
  }
}

// U [L][N] row-major -> U^T [N][Lp] zero-padded (global path)
template <typename T>
__global__ void transpose_pad_kernel(const double* __restrict__ U, double* __restrict__ Ut, int L, int N, int Lp) {
  __shared__ T tile[32][33];
  const T* src = reinterpret_cast<const T*>(U);
  T* dst = reinterpret_cast<T*>(Ut);
  const int x0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const int x = x0 + dy, c = c0 + threadIdx.x;
    T v;
    if (x < L && c < N) v = src[(size_t)x * N + c];
    else v = Sc<T>::zero();
    tile[dy][threadIdx.x] = v;
  }
  __syncthreads();
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const int c = c0 + dy, x = x0 + threadIdx.x;
    if (c < N && x < Lp) dst[(size_t)c * Lp + x] = tile[threadIdx.x][dy];
  }
}

}  // namespace ffsk
