#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, double b, int n) {
  double x = a, y = b;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, b, a);
  t1 = clock64(); cyc[0] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dadd_rn(x, b);
  t1 = clock64(); cyc[1] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dmul_rn(x, b);
  t1 = clock64(); cyc[2] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __ddiv_rn(x, b);
  t1 = clock64(); cyc[3] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x + a);
  t1 = clock64(); cyc[4] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1);
  t1 = clock64(); cyc[5] = t1 - t0;
  float f = (float)a;
  t0 = clock64();
  for (int i = 0; i < n; ++i) f = fmaf(f, (float)b, (float)a);
  t1 = clock64(); cyc[6] = t1 - t0;
  out[threadIdx.x] = x + y + f;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 64); cudaMallocManaged(&c, 8 * 8);
  for (int r = 0; r < 2; ++r) { k<<<1, 32>>>(o, c, 1.0000001, 0.9999999, 1000); cudaDeviceSynchronize(); }
  const char* nm[] = {"dfma", "dadd", "dmul", "ddiv_rn", "dsqrt", "shfl+dadd", "ffma"};
  for (int i = 0; i < 7; ++i) printf("%s %.1f cycles/op\n", nm[i], c[i] / 1000.0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0); printf("clock attr %d kHz\n", clk);
}
