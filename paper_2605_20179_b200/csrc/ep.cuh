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
#include "route.cuh"

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


// ---------------------------------------------------------------- peer-memory EP
// tide_ctx_create_ep_p2p: the same EP step with the two exchanges done by the kernels
// themselves over peer memory (NVLink / NVSwitch P2P stores into the other ranks'
// symmetric regions, counter arrivals with release semantics) instead of NCCL collectives:
//   route kernel (route.cuh) dispatch fused into the router: X rows, top-k ids, gates and
//                           the token count go straight into every rank's x_all /
//                           topk_all / gates_all / ntok at [rank*maxN + n]; one arrival per
//                           source rank on each destination's dispatch counter
//                           the route grid's last CTA then waits until all P sources have
//                           arrived and builds the local experts' token lists (route_ep_lists)
//   tide_ffn_kernel<T,true> (p2p) the phase-2 epilogue stores each routed pair's y row
//                           straight into the owning rank's ypair[n*k + j]; the grid's last
//                           CTA delivers the local experts' counts into every hits_all and
//                           arrives once per rank on its combine counter (ffn.cuh)
//   tide_ep_final_kernel    (p2p) waits for the P arrivals, then exactly the single-device
//                           combine: out[n] = sum_j g[n,j] y[n,j] in slot order (+ shared),
//                           so the EP output equals the single-device output bit for bit
// Counters are double-buffered by the step parity word the route kernel flips; the route's
// list build of a step zeroes the other parity's counters (their last readers finished a
// step ago; their next writers need this step's partials first).  A waiting CTA gives up after
// kEpWaitNs, records the failure in the context's error word and returns (no GPU hang).
constexpr int kEpMaxWorld = 8;
constexpr unsigned long long kEpWaitNs = 20000000000ull;  // 20 s

struct EpPeers {
  char* base[kEpMaxWorld];  // symmetric region of every rank (own included), rank order
};

static_assert(kEpMaxWorld == kRouteEpMax, "route.cuh and ep.cuh disagree on the max world");

struct EpSymLayout {  // byte offsets inside a rank's symmetric region
  size_t x_all, cnt_l, list_l, dst_l, ypair, hits_all, ctr, total;
  // x_all: [P * maxN][H] token rows dispatched by every source rank (row src * maxN + n)
  // cnt_l: [2][El] local-expert counts by step parity, appended to by every source's router
  // list_l / dst_l: [El][P * maxN] x_all row / (source rank << 28 | pair row) of each slot
  // ypair: [maxN * k][H] fp32, y of this rank's pair (n, j) written by its expert's owner
  // ctr: [0..1] dispatch arrivals by parity, [2..3] combine arrivals by parity, [4] error
};

__device__ __forceinline__ unsigned ld_acquire_sys_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_sys_add_u32(unsigned* p, unsigned v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Thread 0 spins until *ctr >= target (acquire, system scope); the CTA then proceeds.
// Returns false (for every thread) on timeout, after recording it in *err.
__device__ __forceinline__ bool ep_wait_all(const unsigned* ctr, unsigned target, unsigned* err) {
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    int ok = 1;
    if (ld_acquire_sys_u32(ctr) < target) {
      const unsigned long long t0 = globaltimer_ns();
      while (ld_acquire_sys_u32(ctr) < target) {
        __nanosleep(128);
        if (globaltimer_ns() - t0 > kEpWaitNs) {
          atomicExch(err, 1u);
          ok = 0;
          break;
        }
      }
    }
    s_ok = ok;
  }
  __syncthreads();
  return s_ok != 0;
}

// p2p variant of tide_ep_final_kernel: grid (max(N,1), ceil(H/512)), 128 threads x 4 columns.
// Waits for the P ranks' FFN arrivals, then the single-device combine's arithmetic on the
// pairs' y rows in ypair (slot order, fp32 fma, + shared expert, one rounding).  CTA (0,0)
// also copies the global hits.
template <typename T>
__global__ void __launch_bounds__(128) tide_ep_final_p2p_kernel(
    char* sym, EpSymLayout lay, const int* par_word, unsigned target, const float* __restrict__ gates,
    const float* __restrict__ y, T* __restrict__ out, int32_t* __restrict__ hit_counts, int E,
    int N, int k, int H, int shared_row0) {
  pdl_wait();
  pdl_trigger();
  unsigned* ctr = reinterpret_cast<unsigned*>(sym + lay.ctr);
  const int par = __ldcg(par_word);
  const int n = blockIdx.x, lane = threadIdx.x & 31;
  if (n >= N && !(n == 0 && blockIdx.y == 0)) return;
  // world 1 (target 0): the FFN grid this kernel waited on above is the only producer
  if (target > 0 && !ep_wait_all(ctr + 2 + par, target, ctr + 4)) return;
  if (n == 0 && blockIdx.y == 0) {
    const int* hits = reinterpret_cast<const int*>(sym + lay.hits_all);
    for (int i = threadIdx.x; i < E; i += blockDim.x) hit_counts[i] = __ldcg(hits + i);
  }
  if (n >= N) return;
  const float* yp = reinterpret_cast<const float*>(sym + lay.ypair);
  const int c = (blockIdx.y * blockDim.x + threadIdx.x) * 4;
  float g_j = 0.f;
  if (lane < k) g_j = __ldcg(gates + (size_t)n * k + lane);
  const bool valid = c < H;
  const int cc = valid ? c : 0;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 8
  for (int j = 0; j < k; ++j) {
    const float g = __shfl_sync(0xffffffffu, g_j, j);
    const float4 v = __ldcg(reinterpret_cast<const float4*>(yp + ((size_t)n * k + j) * H + cc));
    acc.x = fmaf(g, v.x, acc.x);
    acc.y = fmaf(g, v.y, acc.y);
    acc.z = fmaf(g, v.z, acc.z);
    acc.w = fmaf(g, v.w, acc.w);
  }
  if (!valid) return;
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
