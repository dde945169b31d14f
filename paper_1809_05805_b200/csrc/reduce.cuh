// Deterministic grid reductions: per-CTA partials, last-CTA fixed-order sum.
#pragma once
#include "common.cuh"

namespace lsb {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

// Block-reduce NE per-thread values (op: 0 = sum, 1 = max), write the CTA's
// partials entry-major (partial[e*gridDim.x + cta]), and let the last CTA to
// arrive produce out[e] by a fixed-order tree over CTAs.  Every thread of
// the block must call it.  Returns true in the CTA that finalised.
template <int NE>
__device__ bool grid_reduce(const double (&v)[NE], const int (&op)[NE], double* partial,
                            unsigned* counter, double* out) {
  __shared__ double red[kWarps][NE];
  __shared__ bool is_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    double x = op[e] ? warp_max(v[e]) : warp_sum(v[e]);
    if (lane == 0) red[warp][e] = x;
  }
  __syncthreads();
  if (threadIdx.x < NE) {
    const int e = threadIdx.x;
    double x = red[0][e];
    for (int w = 1; w < kWarps; ++w) x = op[e] ? fmax(x, red[w][e]) : x + red[w][e];
    partial[(size_t)e * gridDim.x + blockIdx.x] = x;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = atomicAdd(counter, 1u);
    is_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last) return false;
  __threadfence();
  const int G = gridDim.x;
  for (int e = warp; e < NE; e += kWarps) {
    double x = op[e] ? 0.0 : 0.0;
    bool first = true;
    for (int c = lane; c < G; c += 32) {
      double y = __ldcg(partial + (size_t)e * G + c);
      if (first) { x = y; first = false; } else { x = op[e] ? fmax(x, y) : x + y; }
    }
    if (first) x = op[e] ? 0.0 : 0.0;
    x = op[e] ? warp_max(x) : warp_sum(x);
    if (lane == 0) out[e] = x;
  }
  if (threadIdx.x == 0) *counter = 0u;
  return true;
}

}  // namespace lsb
