// analytics.cuh -- NEXT-4: routing-trace analytics on the GPU.
//   tide_trace_sim_kernel    sim[s][t] = cos(c_s, c_t) of per-step hit-count vectors
//                            (integer dot products are exact in int64; one fp64 division)
//   tide_trace_step_kernel   unique experts per step; drift d_t = |topB(t) \ topB(t-1)| / B
//                            (Eq. 4; top-B by (hits desc, id asc) as a4)
#pragma once
#include "ptx.cuh"

namespace tide {

// grid (T, T), 256 threads
__global__ void __launch_bounds__(256) tide_trace_sim_kernel(const int* __restrict__ counts,
                                                             int T, int E,
                                                             double* __restrict__ sim) {
  const int s = blockIdx.x, t = blockIdx.y;
  long long ab = 0, aa = 0, bb = 0;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const long long a = counts[(size_t)s * E + e], b = counts[(size_t)t * E + e];
    ab += a * b;
    aa += a * a;
    bb += b * b;
  }
  __shared__ long long red[3][8];
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    ab += __shfl_xor_sync(0xffffffffu, ab, o);
    aa += __shfl_xor_sync(0xffffffffu, aa, o);
    bb += __shfl_xor_sync(0xffffffffu, bb, o);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { red[0][warp] = ab; red[1][warp] = aa; red[2][warp] = bb; }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long x = 0, y = 0, z = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { x += red[0][w]; y += red[1][w]; z += red[2][w]; }
    sim[(size_t)s * T + t] = (y == 0 || z == 0) ? 0.0 : (double)x / (sqrt((double)y) * sqrt((double)z));
  }
}

// grid T, 1024 threads; dynamic smem 2 * E bytes
__global__ void __launch_bounds__(1024) tide_trace_step_kernel(const int* __restrict__ counts,
                                                               int T, int E, int B,
                                                               int* __restrict__ unique,
                                                               double* __restrict__ drift) {
  extern __shared__ uint8_t in_b[];  // [2][E]: top-B membership of steps t-1 and t
  __shared__ int s_u, s_d;
  const int t = blockIdx.x;
  if (threadIdx.x == 0) { s_u = 0; s_d = 0; }
  __syncthreads();
  for (int q = 0; q < 2; ++q) {
    const int st = t - 1 + q;
    if (st < 0) continue;
    const int* c = counts + (size_t)st * E;
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
      const int he = c[e];
      int r = 0;
      for (int f = 0; f < E; ++f) {
        const int hf = c[f];
        r += (hf > he) || (hf == he && f < e);
      }
      in_b[q * E + e] = r < B;
      if (q == 1 && he > 0) atomicAdd(&s_u, 1);
    }
  }
  __syncthreads();
  if (t > 0)
    for (int e = threadIdx.x; e < E; e += blockDim.x)
      if (in_b[E + e] && !in_b[e]) atomicAdd(&s_d, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    unique[t] = s_u;
    if (t > 0) drift[t - 1] = (double)s_d / (double)B;
  }
}

}  // namespace tide
