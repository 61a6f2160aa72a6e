// Host-side helpers shared by the translation units of libffs.so (ffs_abi.cu and the extension
// calls of ffs_ext.cu): error reporting, launch accounting, tuning options, plan helpers and the
// measurement hooks. Defined in ffs_abi.cu.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace ffsh {

// ffs_last_error() message for the current thread; returns `code`
int fail(int code, const char* fmt, ...);
void clear_error();

// kernel launches of the last sampling call on this thread (ffs_last_launch_count)
int& launches();

// tuning options (ffs_set_option); process-wide, read when a plan is made
double option(int opt);
uint64_t options_version();

// current device and its SM count (cached per device)
int device();
int sm_count(int dev);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize = 227 KB) once per kernel and device, so that
// cached plans of any shared-memory size can launch the kernel
int ensure_max_smem(const void* fn);

constexpr size_t kAlign = 256;
inline size_t align_up(size_t v) { return (v + kAlign - 1) & ~(kAlign - 1); }
constexpr size_t kMaxSmem = 227 * 1024;

// measurement hooks (ffs_profile_enable): events around the dominant kernel(s) of a call
bool profiling();
void prof_begin(cudaStream_t s);
void prof_end(cudaStream_t s);

}  // namespace ffsh
