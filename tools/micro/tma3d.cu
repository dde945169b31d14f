// One 3-D tensor copy (cp.async.bulk.tensor, OOB zero fill) of a box of
// doubles into shared memory, copied back out: checks the tensor-map
// recipe of stencil27_tile_kernel in isolation.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/tma3d tools/micro/tma3d.cu && /tmp/tma3d
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__global__ void k(const __grid_constant__ CUtensorMap tm, double* out, int c0, int c1, int c2,
                  int nbox) {
  extern __shared__ __align__(128) unsigned char raw[];
  double* s = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(raw) + 127) & ~(uintptr_t)127);
  __shared__ uint64_t bar;
  const unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(nbox * 8)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"((unsigned)__cvta_generic_to_shared(s)),
        "l"(reinterpret_cast<uint64_t>(&tm)), "r"(c0), "r"(c1), "r"(c2), "r"(b)
        : "memory");
  }
  unsigned done = 0;
  while (!done)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(b)
        : "memory");
  for (int i = threadIdx.x; i < nbox; i += blockDim.x) out[i] = s[i];
}

typedef CUresult (*enc_fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                           const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                           CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                           CUtensorMapFloatOOBfill);

static int run(int nx, int ny, int nz, int bx, int by, int c0, int c1, int c2, int l2) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  enc_fn enc = (enc_fn)p;
  const size_t n = (size_t)nx * ny * nz;
  double *x, *out;
  cudaMalloc(&x, n * 8);
  cudaMalloc(&out, (size_t)bx * by * 8);
  double* h = (double*)malloc(n * 8);
  for (size_t i = 0; i < n; ++i) h[i] = (double)i + 1;
  cudaMemcpy(x, h, n * 8, cudaMemcpyHostToDevice);
  CUtensorMap tm;
  const cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz};
  const cuuint64_t str[2] = {(cuuint64_t)nx * 8, (cuuint64_t)nx * ny * 8};
  const cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, x, dims, str, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   (CUtensorMapL2promotion)l2, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  k<<<1, 128, bx * by * 8 + 256>>>(tm, out, c0, c1, c2, bx * by);
  cudaError_t e = cudaDeviceSynchronize();
  int bad = 0;
  if (e == cudaSuccess) {
    double* o = (double*)malloc((size_t)bx * by * 8);
    cudaMemcpy(o, out, (size_t)bx * by * 8, cudaMemcpyDeviceToHost);
    for (int j = 0; j < by; ++j)
      for (int i = 0; i < bx; ++i) {
        const int gx = c0 + i, gy = c1 + j;
        const bool in = gx >= 0 && gx < nx && gy >= 0 && gy < ny && c2 >= 0 && c2 < nz;
        const double want = in ? h[((size_t)c2 * ny + gy) * nx + gx] : 0.0;
        if (o[j * bx + i] != want) ++bad;
      }
    free(o);
  }
  printf("dims %d %d %d box %d %d at (%d,%d,%d) l2=%d: encode %d, kernel %s, mismatches %d\n", nx,
         ny, nz, bx, by, c0, c1, c2, l2, (int)r, cudaGetErrorString(e), bad);
  cudaFree(x); cudaFree(out); free(h);
  return e == cudaSuccess ? 0 : 1;
}

int main(int argc, char** argv) {
  const int which = argc > 1 ? atoi(argv[1]) : 0;
  switch (which) {
    case 0: return run(64, 32, 8, 16, 8, 0, 0, 1, 0);
    case 1: return run(64, 32, 8, 34, 18, 0, 0, 1, 0);
    case 2: return run(64, 32, 8, 34, 18, -1, -1, 1, 0);
    case 3: return run(64, 32, 8, 34, 18, -1, -1, 1, 3);
    case 4: return run(12, 10, 8, 34, 18, -1, -1, 1, 0);
    case 5: return run(64, 32, 8, 32, 16, 0, 0, 1, 3);
    case 6: return run(64, 32, 8, 36, 18, -2, -1, 1, 0);
  }
  return 0;
}
