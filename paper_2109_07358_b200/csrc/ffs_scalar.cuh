// Scalar arithmetic for the FFS kernels: real fp64 (FFS_F64) and complex128 (FFS_C128).
// Complex products are BILINEAR (u_x^T h; reading Q3): no conjugation anywhere
// except in |z|^2 and in the reciprocal of a pivot.
#pragma once
#include <cstdio>
#include <cuda_runtime.h>

// Device-side bounds checks of the checked build (python -m paper_2109_07358_b200.build --checked
// -> libffs_checked.so, compiled with -DFFS_CHECKED): a failed check prints its condition and
// traps. compute-sanitizer is closed on this GPU pool (profiles/r02/compute_sanitizer_closed.log);
// these checks guard every index the kernels derive from data (sites, permuted columns).
#ifdef FFS_CHECKED
#define FFS_CHECK(cond)                                                                   \
  do {                                                                                    \
    if (!(cond)) {                                                                        \
      printf("FFS_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x);                                          \
      __trap();                                                                           \
    }                                                                                     \
  } while (0)
#else
#define FFS_CHECK(cond) \
  do {                  \
  } while (0)
#endif

struct cplx {
  double re, im;
};

// 1/a to ~1 ulp: hardware approximation + two Newton steps (no slow path; pivots are normal
// numbers — a zero or subnormal pivot only occurs on the flagged degenerate path)
__device__ __forceinline__ double fast_rcp(double a) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
  double e = fma(-a, r, 1.0);
  r = fma(r, e, r);
  e = fma(-a, r, 1.0);
  return fma(r, e, r);
}

template <typename T> struct Sc;

template <> struct Sc<double> {
  static constexpr int kDoubles = 1;
  __device__ __forceinline__ static double zero() { return 0.0; }
  __device__ __forceinline__ static double one() { return 1.0; }
  __device__ __forceinline__ static double neg(double a) { return -a; }
  __device__ __forceinline__ static double add(double a, double b) { return a + b; }
  // c - a*b
  __device__ __forceinline__ static double fms(double a, double b, double c) { return fma(-a, b, c); }
  __device__ __forceinline__ static double mul(double a, double b) { return a * b; }
  __device__ __forceinline__ static double abs2(double a) { return a * a; }
  __device__ __forceinline__ static double recip(double a) { return fast_rcp(a); }
  __device__ __forceinline__ static bool finite(double a) { return isfinite(a); }
};

template <> struct Sc<cplx> {
  static constexpr int kDoubles = 2;
  __device__ __forceinline__ static cplx zero() { return {0.0, 0.0}; }
  __device__ __forceinline__ static cplx one() { return {1.0, 0.0}; }
  __device__ __forceinline__ static cplx neg(cplx a) { return {-a.re, -a.im}; }
  __device__ __forceinline__ static cplx add(cplx a, cplx b) { return {a.re + b.re, a.im + b.im}; }
  __device__ __forceinline__ static cplx fms(cplx a, cplx b, cplx c) {
    cplx r;
    r.re = fma(-a.re, b.re, fma(a.im, b.im, c.re));
    r.im = fma(-a.re, b.im, fma(-a.im, b.re, c.im));
    return r;
  }
  __device__ __forceinline__ static cplx mul(cplx a, cplx b) {
    cplx r;
    r.re = fma(a.re, b.re, -a.im * b.im);
    r.im = fma(a.re, b.im, a.im * b.re);
    return r;
  }
  __device__ __forceinline__ static double abs2(cplx a) { return fma(a.re, a.re, a.im * a.im); }
  __device__ __forceinline__ static cplx recip(cplx a) {
    double d = fast_rcp(fma(a.re, a.re, a.im * a.im));
    return {a.re * d, -a.im * d};
  }
  __device__ __forceinline__ static bool finite(cplx a) { return isfinite(a.re) && isfinite(a.im); }
};
