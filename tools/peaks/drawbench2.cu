// Draw-step latency variants (development): cycles per dependent draw for one warp alone and
// per warp with 12 warps resident on the SM (3 per scheduler, the C2 kernel's occupancy).
//   A  seg_draw<8,32>: 5-level fp64 shuffle scan (the kernel's draw)
//   B  warp_draw_fast<8>: 8-lane group scan + group offsets by shuffle
//   C  4-lane group shuffle scan (2 levels) + 8 group totals through shared memory
//   D  all 32 lane totals through shared memory, every lane sums its prefix and the total
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2109_07358_b200/csrc/ffs_warp_kernel.cuh"
using namespace ffsk;

// C: groups of 4 lanes scanned by shuffles, group totals through smem (8 doubles)
__device__ __forceinline__ Draw draw_c(const double (&col)[8], double u, double* scr) {
  const int lane = threadIdx.x & 31;
  double cs[8];
  cs[0] = col[0] * col[0];
#pragma unroll
  for (int r = 1; r < 8; ++r) cs[r] = fma(col[r], col[r], cs[r - 1]);
  const double tot = cs[7];
  double incl = SegOps<4>::scan_level(tot, 1);
  incl = SegOps<4>::scan_level(incl, 2);
  if ((lane & 3) == 3) scr[lane >> 2] = incl;
  __syncwarp();
  double g[8];
#pragma unroll
  for (int i = 0; i < 8; i += 2) {
    const double2 d = *reinterpret_cast<const double2*>(scr + i);
    g[i] = d.x;
    g[i + 1] = d.y;
  }
  const int q = lane >> 2;
  // exclusive group offset: sum of g[i] for i < q (tree with masks)
  double m[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) m[i] = (i < q) ? g[i] : 0.0;
  const double off = ((m[0] + m[1]) + (m[2] + m[3])) + ((m[4] + m[5]) + (m[6] + m[7]));
  Draw d;
  d.T = ((g[0] + g[1]) + (g[2] + g[3])) + ((g[4] + g[5]) + (g[6] + g[7]));
  const double excl = off + (incl - tot);
  const bool ok = (d.T > 0.0) && (d.T < INFINITY);
  const double tp = fmax(fma(u, d.T, -excl), 0.0);
  d.ball = __ballot_sync(0xffffffffu, ok && (tot > tp));
  int cnt = 0;
#pragma unroll
  for (int r = 0; r < 7; ++r) cnt += (cs[r] <= tp) ? 1 : 0;
  d.rsel = cnt;
  return d;
}

// D: all 32 lane totals through smem; masked tree sums
__device__ __forceinline__ Draw draw_d(const double (&col)[8], double u, double* scr) {
  const int lane = threadIdx.x & 31;
  double cs[8];
  cs[0] = col[0] * col[0];
#pragma unroll
  for (int r = 1; r < 8; ++r) cs[r] = fma(col[r], col[r], cs[r - 1]);
  const double tot = cs[7];
  scr[lane] = tot;
  __syncwarp();
  double tb[4], eb[4];
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    double v[8];
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      const double2 d = *reinterpret_cast<const double2*>(scr + 8 * b + i);
      v[i] = d.x;
      v[i + 1] = d.y;
    }
    double m[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) m[i] = (8 * b + i < lane) ? v[i] : 0.0;
    tb[b] = ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
    eb[b] = ((m[0] + m[1]) + (m[2] + m[3])) + ((m[4] + m[5]) + (m[6] + m[7]));
  }
  Draw d;
  d.T = (tb[0] + tb[1]) + (tb[2] + tb[3]);
  const double excl = (eb[0] + eb[1]) + (eb[2] + eb[3]);
  const bool ok = (d.T > 0.0) && (d.T < INFINITY);
  const double tp = fmax(fma(u, d.T, -excl), 0.0);
  d.ball = __ballot_sync(0xffffffffu, ok && (tot > tp));
  int cnt = 0;
#pragma unroll
  for (int r = 0; r < 7; ++r) cnt += (cs[r] <= tp) ? 1 : 0;
  d.rsel = cnt;
  return d;
}

template <int V>
__global__ void kdraw(double* out, long long* cyc, int iters) {
  __shared__ double scr_all[16][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* scr = scr_all[wid];
  double col[8];
  for (int r = 0; r < 8; ++r) col[r] = 0.01 * (lane * 8 + r + 1);
  double u = 0.37;
  int acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    Draw d;
    if constexpr (V == 0) d = seg_draw<8, 32>(col, u, 0);
    else if constexpr (V == 1) d = warp_draw_fast<8>(col, u, lane);
    else if constexpr (V == 2) d = draw_c(col, u, scr);
    else d = draw_d(col, u, scr);
    const int own = __ffs(d.ball) - 1;
    const int orow = __shfl_sync(0xffffffffu, d.rsel, own);
    acc += orow;
    col[0] += 1e-12 * (orow + own);  // next draw depends on this one
    u = u * 0.999 + 0.0005;
  }
  long long t1 = clock64();
  if (lane == 0) cyc[wid] = (t1 - t0) / iters;
  out[threadIdx.x] = acc + col[0];
}

int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 4096);
  cudaMalloc(&c, 16 * 8);
  const char* names[] = {"A_seg_draw", "B_warp_draw_fast", "C_grp4_smem", "D_smem32"};
  printf("{");
  for (int v = 0; v < 4; ++v) {
    for (int warps : {1, 12}) {
      for (int rep = 0; rep < 2; ++rep) {
        const int it = rep ? 4000 : 100;
        if (v == 0) kdraw<0><<<1, 32 * warps>>>(o, c, it);
        if (v == 1) kdraw<1><<<1, 32 * warps>>>(o, c, it);
        if (v == 2) kdraw<2><<<1, 32 * warps>>>(o, c, it);
        if (v == 3) kdraw<3><<<1, 32 * warps>>>(o, c, it);
      }
      cudaDeviceSynchronize();
      long long h[16];
      cudaMemcpy(h, c, 16 * 8, cudaMemcpyDeviceToHost);
      printf("%s\"%s_w%d\": %lld", (v || warps > 1) ? ", " : "", names[v], warps, h[0]);
    }
  }
  printf("}\n");
  return 0;
}
