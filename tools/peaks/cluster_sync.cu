// Cluster-barrier latency (development): cycles per barrier.cluster arrive.release/wait.acquire
// round for clusters of CS CTAs x T threads, with and without one DSMEM store per CTA per round,
// and per __syncthreads round for comparison.
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>

__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void csync_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}

template <int MODE>
__global__ void kbar(long long* out, int iters) {
  __shared__ double box[32];
  unsigned rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  unsigned ncta;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(ncta));
  if (threadIdx.x < 32) box[threadIdx.x] = 0.0;
  csync();
  long long t0 = clock64();
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    if (MODE == 1 && threadIdx.x < ncta) {
      unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(&box[rank])), ra;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(threadIdx.x));
      asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"((double)it) : "memory");
    }
    if (MODE == 2) __syncthreads();
    else if (MODE == 3) csync_relaxed();
    else csync();
    acc += box[(it + rank) & 7];
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && rank == 0) out[blockIdx.x / ncta] = (t1 - t0) / iters;
  if (acc == -1.0) out[0] = 0;
}

int main() {
  long long* o;
  cudaMalloc(&o, 1024 * 8);
  printf("{");
  bool first = true;
  for (int cs : {2, 4, 8, 16}) {
    for (int mode = 0; mode < 4; ++mode) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs);
      cfg.blockDim = dim3(512);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      void (*fn)(long long*, int) = mode == 0 ? kbar<0> : mode == 1 ? kbar<1> : mode == 2 ? kbar<2> : kbar<3>;
      if (cs > 8) cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaError_t e = cudaLaunchKernelEx(&cfg, fn, o, 2000);
      e = cudaLaunchKernelEx(&cfg, fn, o, 2000);
      cudaDeviceSynchronize();
      long long h = -1;
      if (e == cudaSuccess) cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
      const char* names[] = {"cluster_sync", "cluster_sync+dsmem_store", "syncthreads", "cluster_sync_relaxed"};
      printf("%s\"%s_cs%d\": %lld", first ? "" : ", ", names[mode], cs, h);
      first = false;
    }
  }
  printf("}\n");
  return 0;
}
