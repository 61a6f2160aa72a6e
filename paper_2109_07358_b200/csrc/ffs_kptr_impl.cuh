// Definitions of the kernel-pointer getters of ffs_kptr.h (included by the generated
// per-instantiation translation units, see build.py).
#pragma once
#include "ffs_kptr.h"
#include "ffs_kernel.cuh"
#include "ffs_warp_kernel.cuh"
#include "ffs_cluster_kernel.cuh"

namespace ffsk {
template <typename T, bool WARP, int R, int B, bool USMEM, int MAXT> const void* sample_kernel_ptr() {
  return reinterpret_cast<const void*>(&ffs_sample_kernel<T, WARP, R, B, USMEM, MAXT>);
}
template <int R, int B, int G, int MAXT> const void* seg_kernel_ptr() {
  return reinterpret_cast<const void*>(&ffs_seg_kernel<R, B, G, MAXT>);
}
template <typename T, int R, int B, int MAXT> const void* cluster_kernel_ptr() {
  return reinterpret_cast<const void*>(&ffs_cluster_kernel<T, R, B, MAXT>);
}
template <typename T, int R, int B, int MAXT> const void* cluster_step_kernel_ptr() {
  return reinterpret_cast<const void*>(&ffs_cluster_kernel<T, R, B, MAXT, true>);
}
}  // namespace ffsk
