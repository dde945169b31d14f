// st.async + mbarrier complete_tx handoff between CTAs of a cluster:
// ranks 1..C-1 push a 16-byte value per "iteration" into rank 0's shared
// memory counted on rank 0's mbarrier; rank 0 pushes back into every rank's
// barrier.  Checks the values and counts cycles per round trip.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa_u32(const void* p, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_v2(uint32_t dst, double a, double b, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];"
               :: "r"(dst), "d"(a), "d"(b), "r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  unsigned done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(smem_u32(b)), "r"(parity) : "memory");
}

__global__ void kern(int iters, long long* out, int* err) {
  cg::cluster_group cl = cg::this_cluster();
  const int rank = cl.block_rank(), cs = cl.num_blocks();
  __shared__ __align__(16) double slots[16][2];
  __shared__ __align__(16) double back[2];
  __shared__ __align__(8) uint64_t mb;
  if (threadIdx.x == 0) {
    mbar_init(&mb, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl.sync();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (rank != 0) {
      if (threadIdx.x == 0) mbar_expect(&mb, 16);                   // arm for the reply
      if (threadIdx.x == 0) st_async_v2(mapa_u32(&slots[rank][0], 0), (double)i, (double)rank, mapa_u32(&mb, 0));
      mbar_wait(&mb, i & 1);
      if (threadIdx.x == 0 && (back[0] != (double)i || back[1] != -1.0)) atomicAdd(err, 1);
    } else {
      if (threadIdx.x == 0) mbar_expect(&mb, 16 * (cs - 1));
      mbar_wait(&mb, i & 1);
      for (int c = 1 + threadIdx.x; c < cs; c += blockDim.x) {
        if (slots[c][0] != (double)i || slots[c][1] != (double)c) atomicAdd(err, 1);
        st_async_v2(mapa_u32(back, c), (double)i, -1.0, mapa_u32(&mb, c));
      }
    }
  }
  long long t1 = clock64();
  cl.sync();
  if (threadIdx.x == 0 && rank == 1) out[0] = (t1 - t0) / iters;
}

int main() {
  long long* o; int* e;
  cudaMallocManaged(&o, 8); cudaMallocManaged(&e, 4); *e = 0;
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {2, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs); cfg.blockDim = dim3(128);
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, 1000, o, e);
    cudaError_t r = cudaDeviceSynchronize();
    printf("cluster %2d: %lld cycles per push+reply round trip, errors %d (%s)\n", cs, o[0], *e, cudaGetErrorString(r));
  }
}
