// route.cuh -- a1..a5 of the TIDE layer-step:
//   tide_router_kernel  a1  logits = X Wr^T (fp32 accumulate, blocked order, R-17)
//   tide_route_kernel   a2  softmax + top-k (lowest id on ties, R-3/R-4)
//                       a3  hit histogram (shared-memory atomics)
//                       a4  refresh (step % interval == 0) + top-C placement (R-6/R-8)
//                       a5  bucket order / offsets / pos (R-11) + FFN work list + miss list
//   tide_gather_kernel  a5  X_perm[pos[n,j]] = X[n] (and the shared expert's rows)
//   tide_combine_kernel a10 out[n] = sum_j g[n,j] y[pos[n,j]] (+ y_shared[n]), slot order
#pragma once
#include "ptx.cuh"

namespace tide {

constexpr int kRouterWarps = 8;    // experts per router CTA
constexpr int kRouterTokens = 32;  // tokens per router CTA
constexpr int kRouteThreads = 1024;
constexpr int kMaxTok = 128;       // tokens per FFN work entry (MMA N <= 128 + gate/up in TMEM)

// ---------------------------------------------------------------- a1 router
template <typename T>
__device__ __forceinline__ float dot16B(uint4 xa, uint4 wa, float acc);
template <>
__device__ __forceinline__ float dot16B<__nv_bfloat16>(uint4 xa, uint4 wa, float acc) {
  const __nv_bfloat162* x2 = reinterpret_cast<const __nv_bfloat162*>(&xa);
  const __nv_bfloat162* w2 = reinterpret_cast<const __nv_bfloat162*>(&wa);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 xf = __bfloat1622float2(x2[i]);
    float2 wf = __bfloat1622float2(w2[i]);
    acc = fmaf(xf.x, wf.x, acc);
    acc = fmaf(xf.y, wf.y, acc);
  }
  return acc;
}
template <>
__device__ __forceinline__ float dot16B<float>(uint4 xa, uint4 wa, float acc) {
  acc = fmaf(__uint_as_float(xa.x), __uint_as_float(wa.x), acc);
  acc = fmaf(__uint_as_float(xa.y), __uint_as_float(wa.y), acc);
  acc = fmaf(__uint_as_float(xa.z), __uint_as_float(wa.z), acc);
  acc = fmaf(__uint_as_float(xa.w), __uint_as_float(wa.w), acc);
  return acc;
}

// grid (ceil(E/8), ceil(N/32)), 256 threads; dynamic smem = 8 * H * sizeof(T).
// Warp w owns expert e = 8*blockIdx.x + w; its router row is staged in smem once.
// Lane l accumulates 16-byte chunks l, l+32, ... sequentially in fp32, then a
// butterfly over the 32 lane partials (every lane ends with identical bits).
template <typename T>
__global__ void __launch_bounds__(256) tide_router_kernel(const T* __restrict__ x,
                                                          const T* __restrict__ wr,
                                                          float* __restrict__ logits, int N, int E,
                                                          int H) {
  extern __shared__ __align__(16) unsigned char router_smem[];
  uint4* w_s = reinterpret_cast<uint4*>(router_smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int e0 = blockIdx.x * kRouterWarps;
  const int chunks = H * (int)sizeof(T) / 16;
  const int rows = min(kRouterWarps, E - e0);
  for (int i = threadIdx.x; i < rows * chunks; i += blockDim.x)
    w_s[i] = __ldg(reinterpret_cast<const uint4*>(wr + (size_t)e0 * H) + i);
  __syncthreads();
  const int e = e0 + warp;
  if (e >= E) return;
  const uint4* wrow = w_s + warp * chunks;
  const int n0 = blockIdx.y * kRouterTokens, n1 = min(N, n0 + kRouterTokens);
  for (int n = n0; n < n1; ++n) {
    const uint4* xrow = reinterpret_cast<const uint4*>(x + (size_t)n * H);
    float acc = 0.f;
    for (int c = lane; c < chunks; c += 32) acc = dot16B<T>(__ldg(xrow + c), wrow[c], acc);
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) logits[(size_t)n * E + e] = acc;
  }
}

// ---------------------------------------------------------------- a2..a5 route
// Info block written for the host (one D2H copy in host_master mode).
struct RouteInfo {
  int status;          // 0 ok, 3 = TIDE_EPLACEMENT
  int n_entries;       // routed FFN entries (loaded experts + shared expert)
  int n_miss;          // hit experts not loaded in HBM
  int refreshed;
  int promotions, evictions, resident_pairs, unique_experts;
  int sched;           // FFN work counter (zeroed here)
  int pad[7];
  // followed by: miss_e[E], miss_off[E], miss_m[E], hits[E] (int32), placement_out[E] (u8)
};

struct RouteParams {
  const float* logits;
  const uint8_t* placement_in;
  const int* slot_of;   // [E] pool slot of each expert, -1 if not in HBM; nullptr: all in HBM (slot = e)
  int N, E, k, norm_topk, refresh, capacity, shared;
  int* topk_idx;        // [N,k]
  float* gates;         // [N,k]
  int* pos;             // [N,k]
  int* order;           // [E]
  int* offsets;         // [E+1]
  int* hit_counts;      // [E] caller buffer
  uint8_t* placement_out;  // [E] caller buffer
  RouteInfo* info;      // info block (+ trailing arrays)
  int4* entries;        // FFN work list {slot, row offset, tokens, flags}
  int* done;            // per-entry phase-1 completion counters (zeroed here)
};

__device__ __forceinline__ bool better(float va, int ia, float vb, int ib) {
  return va > vb || (va == vb && ia < ib);
}

// Block-wide exclusive scan of one int per thread (blockDim == 1024).
__device__ __forceinline__ int block_excl_scan(int v, int* warp_sums, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) warp_sums[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int s = warp_sums[lane];
    int si = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, si, o);
      if (lane >= o) si += t;
    }
    warp_sums[lane] = si - s;  // exclusive warp prefix
    if (lane == 31) *total = si;
  }
  __syncthreads();
  int r = warp_sums[warp] + incl - v;
  __syncthreads();
  return r;
}

// One CTA of 1024 threads.  E <= 1024, N <= 1024, k <= 32.
// dynamic smem: hits[E] + bstart[E] + order[E] + pl[E](int) + mask[E * NW] (NW = ceil(N/32))
__global__ void __launch_bounds__(kRouteThreads, 1) tide_route_kernel(const RouteParams p) {
  extern __shared__ __align__(16) int route_smem[];
  const int E = p.E, N = p.N, k = p.k;
  const int NW = (N + 31) >> 5;
  int* hits = route_smem;
  int* bstart = hits + E;
  int* order = bstart + E;
  int* pl = order + E;
  unsigned* mask = reinterpret_cast<unsigned*>(pl + E);
  __shared__ int warp_sums[32];
  __shared__ int s_total, s_cnt, s_prom, s_evic;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  for (int i = tid; i < E; i += blockDim.x) hits[i] = 0;
  for (int i = tid; i < E * NW; i += blockDim.x) mask[i] = 0u;
  if (tid == 0) { s_cnt = 0; s_prom = 0; s_evic = 0; }
  __syncthreads();

  // ---- a2: per-token top-k by k rounds of a warp argmax (value desc, id asc)
  const int epl = (E + 31) >> 5;  // logits per lane
  for (int n = warp; n < N; n += 32) {
    float v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int e = lane + 32 * i;
      v[i] = (i < epl && e < E) ? p.logits[(size_t)n * E + e] : -INFINITY;
    }
    unsigned taken = 0u;
    int my_e = 0;
    float my_l = 0.f;
    for (int j = 0; j < k; ++j) {
      float bv = -INFINITY;
      int bi = 0x7fffffff;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int e = lane + 32 * i;
        if (i < epl && e < E && !((taken >> i) & 1u) && better(v[i], e, bv, bi)) {
          bv = v[i];
          bi = e;
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (better(ov, oi, bv, bi)) { bv = ov; bi = oi; }
      }
      if ((bi & 31) == lane) taken |= 1u << (bi >> 5);
      if (lane == j) { my_e = bi; my_l = bv; }
    }
    // gates (R-2): softmax probabilities of the selected experts, renormalised or not
    const float m = __shfl_sync(0xffffffffu, my_l, 0);  // top-1 logit = max
    float denom;
    if (p.norm_topk) {
      float t = lane < k ? expf(my_l - m) : 0.f;
#pragma unroll
      for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      denom = t;
    } else {
      float z = 0.f;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int e = lane + 32 * i;
        if (i < epl && e < E) z += expf(v[i] - m);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
      denom = z;
    }
    if (lane < k) {
      p.topk_idx[(size_t)n * k + lane] = my_e;
      p.gates[(size_t)n * k + lane] = expf(my_l - m) / denom;
      atomicAdd(&hits[my_e], 1);                                   // a3
      atomicOr(&mask[my_e * NW + (n >> 5)], 1u << (n & 31));
    }
  }
  __syncthreads();

  // ---- a4: refresh -> top-C by (hits desc, id asc); otherwise keep the input placement
  for (int e = tid; e < E; e += blockDim.x) {
    int res;
    const int he = hits[e];
    if (p.refresh) {
      int rank = 0;
      for (int f = 0; f < E; ++f) {
        const int hf = hits[f];
        rank += (hf > he) || (hf == he && f < e);
      }
      res = rank < p.capacity;
    } else {
      res = p.placement_in[e] != 0;
      if (res) atomicAdd(&s_cnt, 1);
    }
    pl[e] = res;
    const int was = p.placement_in[e] != 0;
    if (res && !was) atomicAdd(&s_prom, 1);
    if (was && !res) atomicAdd(&s_evic, 1);
    p.hit_counts[e] = he;
  }
  __syncthreads();
  int* info_arr = reinterpret_cast<int*>(p.info + 1);
  int* miss_e = info_arr;
  int* miss_off = miss_e + E;
  int* miss_m = miss_off + E;
  int* info_hits = miss_m + E;
  uint8_t* info_pl = reinterpret_cast<uint8_t*>(info_hits + E);
  if (!p.refresh && s_cnt > p.capacity) {  // S:49, S:263 budget safety
    if (tid == 0) {
      p.info->status = 3;
      p.info->n_entries = 0;
      p.info->n_miss = 0;
      p.info->sched = 0;
    }
    return;
  }

  // ---- a5: bucket order (resident ascending id, then non-resident ascending id)
  const int e = tid;
  const int res = (e < E) ? pl[e] : 0;
  const int res_before = block_excl_scan(res, warp_sums, &s_total);
  const int n_res = s_total;
  if (e < E) {
    const int b = res ? res_before : n_res + (e - res_before);
    order[b] = e;
    p.placement_out[e] = (uint8_t)res;
    info_pl[e] = (uint8_t)res;
    info_hits[e] = hits[e];
  }
  __syncthreads();
  // offsets over bucket positions
  const int be = (tid < E) ? order[tid] : 0;
  const int m_b = (tid < E) ? hits[be] : 0;
  const int off_b = block_excl_scan(m_b, warp_sums, &s_total);
  if (tid < E) {
    bstart[be] = off_b;
    p.order[tid] = be;
    p.offsets[tid] = off_b;
  }
  if (tid == 0) p.offsets[E] = N * k;
  // FFN entries (loaded experts, <= kMaxTok tokens each) and the miss list
  int slot = be;
  if (p.slot_of && tid < E) slot = p.slot_of[be];
  const bool loaded = slot >= 0;
  const int nent = (tid < E && m_b > 0 && loaded) ? (m_b + kMaxTok - 1) / kMaxTok : 0;
  const int is_miss = (tid < E && m_b > 0 && !loaded) ? 1 : 0;
  const int ent_off = block_excl_scan(nent, warp_sums, &s_total);
  const int n_ent_routed = s_total;
  const int miss_idx = block_excl_scan(is_miss, warp_sums, &s_total);
  const int n_miss = s_total;
  for (int c = 0; c < nent; ++c) {
    p.entries[ent_off + c] = make_int4(slot, off_b + c * kMaxTok, min(kMaxTok, m_b - c * kMaxTok), 0);
    p.done[ent_off + c] = 0;
  }
  if (is_miss) {
    miss_e[miss_idx] = be;
    miss_off[miss_idx] = off_b;
    miss_m[miss_idx] = m_b;
  }
  const int n_sh = p.shared ? (N + kMaxTok - 1) / kMaxTok : 0;
  if (tid < n_sh) {
    p.entries[n_ent_routed + tid] =
        make_int4(0, N * k + tid * kMaxTok, min(kMaxTok, N - tid * kMaxTok), 1);
    p.done[n_ent_routed + tid] = 0;
  }
  // resident pairs / unique experts
  const int rp = (tid < E && pl[be]) ? m_b : 0;
  const int uq = (tid < E && m_b > 0) ? 1 : 0;
  __syncthreads();
  block_excl_scan(rp, warp_sums, &s_total);
  const int resident_pairs = s_total;
  block_excl_scan(uq, warp_sums, &s_total);
  if (tid == 0) {
    p.info->status = 0;
    p.info->n_entries = n_ent_routed + n_sh;
    p.info->n_miss = n_miss;
    p.info->refreshed = p.refresh;
    p.info->promotions = s_prom;
    p.info->evictions = s_evic;
    p.info->resident_pairs = resident_pairs;
    p.info->unique_experts = s_total;
    p.info->sched = 0;
  }
  // pos[n,j] = bucket start of its expert + lower tokens that chose the same expert
  for (int q = tid; q < N * k; q += blockDim.x) {
    const int n = q / k;
    const int ee = p.topk_idx[q];
    const unsigned* mk = mask + ee * NW;
    int before = 0;
    for (int w = 0; w < (n >> 5); ++w) before += __popc(mk[w]);
    before += __popc(mk[n >> 5] & ((1u << (n & 31)) - 1u));
    p.pos[q] = bstart[ee] + before;
  }
}

// ---------------------------------------------------------------- a5 gather
// grid N, 256 threads: X_perm[pos[n,j]] = X[n]; shared expert rows X_perm[N*k + n] = X[n].
template <typename T>
__global__ void __launch_bounds__(256) tide_gather_kernel(const T* __restrict__ x,
                                                          const int* __restrict__ pos,
                                                          const RouteInfo* __restrict__ info,
                                                          T* __restrict__ x_perm, int N, int k,
                                                          int H, int shared) {
  if (info->status != 0) return;
  const int n = blockIdx.x;
  const int chunks = H * (int)sizeof(T) / 16;
  const uint4* src = reinterpret_cast<const uint4*>(x + (size_t)n * H);
  __shared__ int rows[33];
  if (threadIdx.x < k) rows[threadIdx.x] = pos[(size_t)n * k + threadIdx.x];
  if (threadIdx.x == 0) rows[k] = N * k + n;
  __syncthreads();
  const int nrows = k + (shared ? 1 : 0);
  for (int c = threadIdx.x; c < chunks; c += blockDim.x) {
    const uint4 v = __ldg(src + c);
    for (int j = 0; j < nrows; ++j)
      reinterpret_cast<uint4*>(x_perm + (size_t)rows[j] * H)[c] = v;
  }
}

// ---------------------------------------------------------------- a10 combine
// grid (N, ceil(H / 1024)), 256 threads x 4 columns.  fp32 FMA over j in slot order
// (then the shared expert), one rounding to the output dtype (R-14).
template <typename T>
__global__ void __launch_bounds__(256) tide_combine_kernel(const float* __restrict__ y,
                                                           const float* __restrict__ gates,
                                                           const int* __restrict__ pos,
                                                           const RouteInfo* __restrict__ info,
                                                           T* __restrict__ out, int N, int k, int H,
                                                           int shared) {
  if (info->status != 0) return;
  const int n = blockIdx.x;
  const int c = (blockIdx.y * blockDim.x + threadIdx.x) * 4;
  if (c >= H) return;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int j = 0; j < k; ++j) {
    const float g = __ldg(gates + (size_t)n * k + j);
    const int r = __ldg(pos + (size_t)n * k + j);
    const float4 v = __ldg(reinterpret_cast<const float4*>(y + (size_t)r * H + c));
    acc.x = fmaf(g, v.x, acc.x);
    acc.y = fmaf(g, v.y, acc.y);
    acc.z = fmaf(g, v.z, acc.z);
    acc.w = fmaf(g, v.w, acc.w);
  }
  if (shared) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(y + (size_t)(N * k + n) * H + c));
    acc.x += v.x;
    acc.y += v.y;
    acc.z += v.z;
    acc.w += v.w;
  }
  T* o = out + (size_t)n * H + c;
  o[0] = from_f32<T>(acc.x);
  o[1] = from_f32<T>(acc.y);
  o[2] = from_f32<T>(acc.z);
  o[3] = from_f32<T>(acc.w);
}

}  // namespace tide
