#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__global__ void kbar(long long* out, int iters, int mode) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double buf[64];
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (mode == 0) {
      asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else if (mode == 1) {
      asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
    } else {
      // with a DSMEM store before the release barrier
      if (threadIdx.x == 0) { double* r = cl.map_shared_rank(buf, 0); r[cl.block_rank()] = i; }
      asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && cl.block_rank() == 0) out[0] = (t1 - t0) / iters;
}
int main() {
  long long* o; cudaMallocManaged(&o, 8);
  cudaFuncSetAttribute(kbar, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int mode = 0; mode < 3; ++mode)
  for (int cs : {2, 4, 8, 16}) {
    for (int threads : {128, 512}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs); cfg.blockDim = dim3(threads); cfg.dynamicSmemBytes = 0;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      for (int r = 0; r < 2; ++r) { cudaLaunchKernelEx(&cfg, kbar, o, 2000, mode); cudaDeviceSynchronize(); }
      printf("mode %d cluster %2d threads %3d: %lld cycles/barrier (%s)\n", mode, cs, threads, o[0], cudaGetErrorString(cudaGetLastError()));
    }
  }
}
