// ep.cuh -- expert-parallel (EP) pieces of the TIDE layer-step (DESIGN R-18).
//
// Rank r of P owns experts [r*El, (r+1)*El), El = E/P.  After the per-rank route kernel:
//   dispatch  : ncclAllGather of the ranks' tokens (x_in), top-k ids and gates
//               (fixed maxN rows per rank, rows >= N_r carry top-k ids -1)
//   tide_ep_lists_kernel   token lists of the local experts over all P*maxN rows
//   tide_ffn_kernel        grouped SwiGLU over the local experts (build mode)
//   tide_ep_partial_kernel per source row: sum_j g_j y_j over the pairs routed to this rank
//                          (fp32, slot order) -> send buffer [P][maxN][H]
//   combine   : ncclAlltoAll of the partials
//   tide_ep_final_kernel   out[n] = sum over ranks in rank order (+ shared expert)
// Hits of the local experts are global (all ranks' tokens); ncclAllGather assembles [E].
#pragma once
#include "ptx.cuh"

namespace tide {

__global__ void __launch_bounds__(256) tide_ep_lists_kernel(const int* __restrict__ topk_all,
                                                            int rows, int k, int e0, int El,
                                                            int* __restrict__ cnt_l,
                                                            int* __restrict__ list_l,
                                                            int list_stride,
                                                            int* __restrict__ pslot_all) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= rows * k) return;
  const int e = topk_all[q];
  if (e >= e0 && e < e0 + El) {
    const int s = atomicAdd(&cnt_l[e - e0], 1);
    list_l[(size_t)(e - e0) * list_stride + s] = q / k;
    pslot_all[q] = s;
  } else {
    pslot_all[q] = -1;
  }
}

// grid (rows, ceil(H/512)), 128 threads x 4 columns.
__global__ void __launch_bounds__(128) tide_ep_partial_kernel(
    const float* __restrict__ y, const int* __restrict__ topk_all,
    const float* __restrict__ gates_all, const int* __restrict__ pslot_all,
    const int* __restrict__ off_l, float* __restrict__ partial, int k, int H, int e0, int El) {
  pdl_wait();
  pdl_trigger();
  const int row = blockIdx.x, lane = threadIdx.x & 31;
  const int c = (blockIdx.y * blockDim.x + threadIdx.x) * 4;
  int r_j = -1;
  float g_j = 0.f;
  if (lane < k) {
    const int q = row * k + lane;
    const int e = __ldcg(topk_all + q);
    if (e >= e0 && e < e0 + El) {
      r_j = __ldcg(off_l + (e - e0)) + __ldcg(pslot_all + q);
      g_j = __ldcg(gates_all + q);
    }
  }
  const bool valid = c < H;
  const int cc = valid ? c : 0;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int j = 0; j < k; ++j) {
    const int r = __shfl_sync(0xffffffffu, r_j, j);
    const float g = __shfl_sync(0xffffffffu, g_j, j);
    if (r < 0) continue;
    const float4 v = __ldcg(reinterpret_cast<const float4*>(y + (size_t)r * H + cc));
    acc.x = fmaf(g, v.x, acc.x);
    acc.y = fmaf(g, v.y, acc.y);
    acc.z = fmaf(g, v.z, acc.z);
    acc.w = fmaf(g, v.w, acc.w);
  }
  if (valid) *reinterpret_cast<float4*>(partial + (size_t)row * H + c) = acc;
}

// grid (N, ceil(H/512)), 128 threads x 4 columns.  recv: [P][maxN][H] fp32.
template <typename T>
__global__ void __launch_bounds__(128) tide_ep_final_kernel(const float* __restrict__ recv,
                                                            const float* __restrict__ y,
                                                            T* __restrict__ out, int P, int maxN,
                                                            int H, int shared_row0) {
  pdl_wait();
  pdl_trigger();
  const int n = blockIdx.x;
  const int c = (blockIdx.y * blockDim.x + threadIdx.x) * 4;
  if (c >= H) return;
  float4 acc = __ldcg(reinterpret_cast<const float4*>(recv + (size_t)n * H + c));
  for (int p = 1; p < P; ++p) {  // rank order
    const float4 v = __ldcg(reinterpret_cast<const float4*>(recv + ((size_t)p * maxN + n) * H + c));
    acc.x += v.x;
    acc.y += v.y;
    acc.z += v.z;
    acc.w += v.w;
  }
  if (shared_row0 >= 0) {
    const float4 v = __ldcg(reinterpret_cast<const float4*>(y + (size_t)(shared_row0 + n) * H + c));
    acc.x += v.x;
    acc.y += v.y;
    acc.z += v.z;
    acc.w += v.w;
  }
  T* o = out + (size_t)n * H + c;
  if constexpr (sizeof(T) == 2) {
    __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x, acc.y), hi = __floats2bfloat162_rn(acc.z, acc.w);
    uint2 pk;
    pk.x = *reinterpret_cast<uint32_t*>(&lo);
    pk.y = *reinterpret_cast<uint32_t*>(&hi);
    *reinterpret_cast<uint2*>(o) = pk;
  } else {
    *reinterpret_cast<float4*>(o) = acc;
  }
}

}  // namespace tide
