// route.cuh -- a1..a5 and a10 of the TIDE layer-step.
//
//   tide_route_kernel  (critical path) one launch, two phases chained by a "last CTA"
//                      counter per token group:
//     phase 1 (all CTAs)   a1  logits = X Wr^T for 8 experts x tpc tokens (fp32, blocked
//                              order, R-17); CTAs of column 0 copy X into x_in (the
//                              FFN gathers its token rows from there)
//     phase 2 (last CTA of each token group)
//                          a2  softmax + top-k (lowest id on ties, R-3/R-4), gates (R-2)
//                          a3  hits: per-expert token counts + token lists (atomics) and
//                              per-expert token bitmasks
//   tide_book_kernel   (off the critical path: concurrent with the FFN)
//                          a4  refresh (step % interval == 0): top-C placement (R-6/R-8)
//                          a5  bucket order (resident first, R-11), offsets, pos, info
//   tide_combine_kernel a10 out[n] = sum_j g[n,j] y[row(n,j)] (+ y_shared[n]), slot order
//
// The FFN's rows are grouped by expert in id order (row of pair (n,j) = off[e] +
// its slot in e's token list); values do not depend on rows, so outputs are bitwise
// independent of the (atomic) arrival order and of placement.
#pragma once
#include "ptx.cuh"

namespace tide {

constexpr int kRouteThreads = 256;  // 8 warps
constexpr int kRouterWarps = 8;     // experts per CTA in phase 1 (one per warp)
constexpr int kMaxTok = 128;        // tokens per FFN work entry (MMA N <= 128)

// ---------------------------------------------------------------- a1 helpers
// Sum of the products of one 16-byte chunk, by a fixed pairwise tree in fp32.  bf16 x bf16
// products are exact in fp32, so the only roundings are the tree's (3 levels for bf16).
// Chunk sums are accumulated in fp64 by the caller (R-17: |logit - fp64| stays ~2e-7 even
// when one feature dominates a lane's sum, e.g. the popularity-bias column).
template <typename T>
__device__ __forceinline__ float chunk_dot(uint4 xa, uint4 wa);
template <>
__device__ __forceinline__ float chunk_dot<__nv_bfloat16>(uint4 xa, uint4 wa) {
  const __nv_bfloat162* x2 = reinterpret_cast<const __nv_bfloat162*>(&xa);
  const __nv_bfloat162* w2 = reinterpret_cast<const __nv_bfloat162*>(&wa);
  float q[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 xf = __bfloat1622float2(x2[i]);
    const float2 wf = __bfloat1622float2(w2[i]);
    q[i] = __fmul_rn(xf.x, wf.x) + __fmul_rn(xf.y, wf.y);
  }
  return (q[0] + q[1]) + (q[2] + q[3]);
}
template <>
__device__ __forceinline__ float chunk_dot<float>(uint4 xa, uint4 wa) {
  return fmaf(__uint_as_float(xa.x), __uint_as_float(wa.x),
              __uint_as_float(xa.y) * __uint_as_float(wa.y)) +
         fmaf(__uint_as_float(xa.z), __uint_as_float(wa.z),
              __uint_as_float(xa.w) * __uint_as_float(wa.w));
}

// Info block written for the host (one D2H copy in host_master mode).
struct RouteInfo {
  int status;          // 0 ok, 3 = TIDE_EPLACEMENT
  int n_entries;       // routed FFN entries (loaded experts + shared expert)
  int n_miss;          // hit experts not loaded in HBM
  int refreshed;
  int promotions, evictions, resident_pairs, unique_experts;
  int pad[8];
  // followed by: hits[E] (int32), placement_out[E] (u8)
};

constexpr int kRouteEpMax = 8;  // == kEpMaxWorld (ep.cuh)

// NEXT-3 cross-layer L2 prefetch of the next layer's likely experts (base == nullptr: off):
// that layer's hit experts at its previous step, in the order its FFN claims them (the shared
// expert first, then ascending id), `span` bytes of each from its start (the gate/up rows).
// A cache hint only: values are unaffected.
constexpr int kPfPiece = 64 * 1024;  // bytes per L2 bulk prefetch
struct L2Prefetch {
  const uint8_t* base;    // next layer's packed experts (device_all)
  const int* list;        // next layer's experts ranked at its previous step
  const int* n;           // number of ranked (hit) experts
  int max;                // budget in experts
  long long xb;           // bytes per packed expert
  long long span;         // bytes prefetched per expert (<= xb)
  const uint8_t* shared;  // nullable: next layer's shared expert (prefetched first)
  long long first;        // pieces [first, max * pieces per expert) of the ranked byte range
};
// Issuer `who` of `nwho` takes pieces who, who + nwho, ... of the byte range (the first-claimed
// experts are covered by the lowest issuers first).
__device__ __forceinline__ void issue_l2_prefetch(const L2Prefetch& f, long long who, long long nwho) {
  if (!f.base) return;
  const int sh = f.shared ? 1 : 0;
  const int n = min(__ldcg(f.n) + sh, f.max);
  const long long ppe = (f.span + kPfPiece - 1) / kPfPiece;
  const long long pieces = (long long)n * ppe;
  for (long long i = f.first + who; i < pieces; i += nwho) {
    const int j = (int)(i / ppe);
    const long long q = (i - (long long)j * ppe) * kPfPiece;
    const uint8_t* src = (j < sh) ? f.shared : f.base + (size_t)__ldcg(f.list + j - sh) * f.xb;
    const uint32_t bytes = (uint32_t)min((long long)kPfPiece, f.span - q);
    prefetch_l2_bulk(src + q, bytes);
  }
}

struct RouteParams {
  const void* x;        // [N,H] caller's block hidden states
  const void* wr;       // [E,H] router
  void* x_in;           // [maxN,H] context copy of X (FFN gather source)
  float* logits;        // [N,E]
  double* logits64;     // [ksplit][maxN][E] fp64 partials over slices of H (TC router, ksplit > 1)
  int ksplit;           // TC router: CTAs per 16-expert tile, each over H / ksplit (1 or 2)
  int N, E, H, k, tpc, norm_topk, maxN;
  int* topk_idx;        // [N,k]
  float* gates;         // [N,k]
  int* pair_slot;       // [N,k] slot of pair (n,j) in its expert's token list
  int* cnt2;            // [2][E] per-expert token counts, double-buffered: this step counts
                        // into cnt2[par] (zero on entry) and zeroes cnt2[par^1] for the next
  int* par;             // device parity word, flipped by the last CTA (so any stream-ordered
                        // or graph-replayed sequence of steps stays consistent)
  int* g_done;          // completion counter of the phase-2 CTAs (self-resetting)
  int* list;            // [E * maxN] tokens of each expert (arrival order)
  unsigned* mask;       // [E * NW] token bitmasks (zeroed by tide_book_kernel)
  int* g_cnt;           // [gridDim.y] completion counters (self-resetting)
  int* zero_i;          // FFN scheduler counters zeroed by CTA (0,0)
  int n_zero;
  unsigned long long* trace;  // debug: 8 timestamps per CTA (nullable)
  // Peer-memory EP dispatch fused into the router (tide_ctx_create_ep_p2p; ep_P == 0: off).
  // Every CTA stores its slice of its token rows of X into every rank's x_all; each token
  // group's phase-2 CTA stores the group's top-k ids and gates; the grid's last CTA stores
  // this rank's token count and arrives (release, system scope) on every rank's dispatch
  // counter for the new parity.  Row of token n of this rank in x_all: ep_rank*maxN + n.
  // Each routed pair (n, j) -> expert e is appended straight into the owning rank's token
  // list of e (owner = e / El): a slot from an atomic on the owner's count, the token's x_all
  // row and the pair's return address in the list -- the owners' lists are complete once
  // every source has arrived, with no list-building pass.
  int ep_P, ep_rank;
  char* ep_base[kRouteEpMax];  // symmetric region of every rank
  size_t ep_off_x, ep_off_ctr;
  size_t ep_off_cnt;           // [2][El] per-parity local-expert counts (this step: [par])
  size_t ep_off_list;          // [El][rows] x_all row of each list slot
  size_t ep_off_dst;           // [El][rows] source rank << 28 | pair row n*k + j of each slot
  int ep_lists, ep_El, ep_rows;  // ep_lists: the grid's last CTA waits for every source
  int ep_shared_dev;           // a peer rank runs on this GPU (one-process emulation or two
                               // processes on one device): the FFN may launch only after the
                               // lists exist (R-22); otherwise it launches early, as without EP
};

struct BookParams {
  const int* cnt;       // [E] hits, or [2][E] selected by par (see RouteParams)
  const int* par;       // nullable: cnt is double-buffered, this step's half = par^1
  int* pf_list;         // nullable (NEXT-3): experts with hits > 0 ranked by (hits desc, id asc)
  int* pf_n;            //   and their number; read by the previous layer's FFN next step
  int pf_by_hits;       //   rank by (hits desc, id asc) instead of by id
  const unsigned* mask; // [E * NW]
  unsigned* mask_rw;    // same, zeroed after use
  const int* topk_idx;  // [N,k]
  const uint8_t* placement_in;
  int N, E, k, refresh, capacity;
  int* acc;             // [E] NEXT-1 counter state (ctx-owned)
  int mode;             // 0 current step (R-5), 1 window since last refresh, 2 cumulative
  int step, incumbent;  // block-relative step; incumbent-aware ties
  int* hit_counts;      // [E] caller buffer
  uint8_t* placement_out;  // [E] caller buffer
  int* order;           // [E]
  int* offsets;         // [E+1]
  int* pos;             // [N,k]
  RouteInfo* info;      // + hits[E] + placement_out[E]
};

__device__ __forceinline__ bool better(float va, int ia, float vb, int ib) {
  return va > vb || (va == vb && ia < ib);
}
// The same order without short-circuit evaluation (predicate logic, no branches).
__device__ __forceinline__ bool better_nb(float va, int ia, float vb, int ib) {
  return (va > vb) | ((va == vb) & (ia < ib));
}
// Order-preserving uint32 key of a float (-0 folded into +0, so key order == float order,
// equal floats <=> equal keys): the warp argmax below runs on redux.sync.
__device__ __forceinline__ unsigned order_key(float v) {
  const unsigned u = __float_as_uint(v + 0.0f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key_value(unsigned k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// In-place exclusive scan of a[0..n) in shared memory by the whole CTA; returns the total.
__device__ __forceinline__ int block_scan_excl(int* a, int n, int* scratch /*33 ints*/) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int b = threadIdx.x * per, e = min(n, b + per);
  int s = 0;
  for (int i = b; i < e; ++i) s += a[i];
  int incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) scratch[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int w = lane < nwarps ? scratch[lane] : 0;
    int wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    scratch[lane] = wi - w;
    if (lane == 31) scratch[32] = wi;
  }
  __syncthreads();
  int run = scratch[warp] + incl - s;
  for (int i = b; i < e; ++i) {
    const int v = a[i];
    a[i] = run;
    run += v;
  }
  const int total = scratch[32];
  __syncthreads();
  return total;
}

// a2 + a3 for token n by one warp.  v_in[i] = logit of expert lane + 32 i.
// Lane l sorts its logits by (value desc, id asc) in registers, then k rounds of a warp
// argmax over the lanes' heads (the winner pops); gates (R-2); per-expert counts, token
// lists and bitmasks by atomics.
template <int EPL>
__device__ __forceinline__ void route_token(const RouteParams& p, int* cnt, int par, int n,
                                            const float (&v_in)[EPL],
                                            unsigned long long* tr = nullptr) {
  const int lane = threadIdx.x & 31;
  const int E = p.E, k = p.k, NW = (p.N + 31) >> 5;
  {
    float v[EPL];
    int id[EPL];
#pragma unroll
    for (int i = 0; i < EPL; ++i) {
      const int e = lane + 32 * i;
      v[i] = e < E ? v_in[i] : -INFINITY;
      id[i] = e;
    }
    // bitonic sorting network over the lane's EPL logits (compile-time indices, branch-free
    // compare-exchanges: the previous bubble sort compiled to one branch per comparison)
#pragma unroll
    for (int kk = 2; kk <= EPL; kk <<= 1)
#pragma unroll
      for (int jj = kk >> 1; jj > 0; jj >>= 1)
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          const int l = i ^ jj;
          if (l > i) {  // compile-time
            const int a = (i & kk) == 0 ? i : l, b = (i & kk) == 0 ? l : i;  // a ranks first
            const bool sw = better_nb(v[b], id[b], v[a], id[a]);
            const float va = v[a], vb = v[b];
            const int ia = id[a], ib = id[b];
            v[a] = sw ? vb : va;
            v[b] = sw ? va : vb;
            id[a] = sw ? ib : ia;
            id[b] = sw ? ia : ib;
          }
        }
    float m = v[0];  // row max
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float z = 0.f;   // full-softmax denominator (norm_topk == 0)
    if (!p.norm_topk) {
#pragma unroll
      for (int i = 0; i < EPL; ++i) z += expf(v[i] - m);
#pragma unroll
      for (int o = 16; o; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
    }
    int my_e = 0;
    float my_l = 0.f;
    for (int j = 0; j < k; ++j) {
      // warp argmax of the lane heads by (value desc, id asc): max key (redux.sync); the lane
      // holding it from a ballot, and only when several lanes hold it (an exact tie) the
      // lowest id among them (a second redux.sync; warp-uniform branch)
      const unsigned hk = order_key(v[0]);
      const unsigned mk = __reduce_max_sync(0xffffffffu, hk);
      const unsigned held = __ballot_sync(0xffffffffu, hk == mk);
      int w = __ffs(held) - 1;
      if (held & (held - 1))
        w = (int)__reduce_min_sync(0xffffffffu, hk == mk ? (unsigned)id[0] : 0xffffffffu) & 31;
      const int bi = __shfl_sync(0xffffffffu, id[0], w);  // off the next round's chain
      if (lane == w) {
#pragma unroll
        for (int i = 0; i + 1 < EPL; ++i) { v[i] = v[i + 1]; id[i] = id[i + 1]; }
        v[EPL - 1] = -INFINITY;
        id[EPL - 1] = 0x7fffffff;
      }
      if (lane == j) { my_e = bi; my_l = key_value(mk); }
    }
    float denom = z;  // gates (R-2)
    if (p.norm_topk) {
      float t = lane < k ? expf(my_l - m) : 0.f;
#pragma unroll
      for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      denom = t;
    }
    if (tr && lane == 0) {  // debug: selection and gates done (after a use of denom)
      if (denom == 1.2345e-30f) tr[7] = 2;
      tr[5] = globaltimer_ns();
    }
    if (lane < k) {
      p.topk_idx[(size_t)n * k + lane] = my_e;
      p.gates[(size_t)n * k + lane] = expf(my_l - m) / denom;
      if (p.ep_P) {  // append the pair to its owner's list of my_e (peer memory)
        const int dst = my_e / p.ep_El, el = my_e - dst * p.ep_El;
        char* b = p.ep_base[dst];
        int* cd = reinterpret_cast<int*>(b + p.ep_off_cnt) + par * p.ep_El + el;
        const int slot = p.ep_P > 1 ? atomicAdd_system(cd, 1) : atomicAdd(cd, 1);
        const size_t q = (size_t)el * p.ep_rows + slot;
        reinterpret_cast<int*>(b + p.ep_off_list)[q] = p.ep_rank * p.maxN + n;
        reinterpret_cast<unsigned*>(b + p.ep_off_dst)[q] =
            ((unsigned)p.ep_rank << 28) | (unsigned)(n * k + lane);
      } else {
        const int slot = atomicAdd(&cnt[my_e], 1);
        p.list[(size_t)my_e * p.maxN + slot] = n;
        p.pair_slot[(size_t)n * k + lane] = slot;
        atomicOr(&p.mask[my_e * NW + (n >> 5)], 1u << (n & 31));
      }
    }
    }
}

// Peer-memory EP, in the route grid's last CTA (after its own arrivals): wait until all P
// sources have dispatched this step (own included) -- their X rows and list appends are then
// in this rank's region -- and free the other parity's dispatch / combine counters for the
// next step (their last readers are done).  A wait that gives up after 20 s records the
// failure in the error word and returns.
__device__ __forceinline__ void route_ep_wait(const RouteParams& p, int par, int& s_last) {
  __shared__ int s_ok;  // the wait's outcome (not s_last: other threads may still be reading it)
  __syncthreads();  // s_last was set by thread 0
  if (!s_last) return;
  if (threadIdx.x == 0) {
    unsigned* ctr = reinterpret_cast<unsigned*>(p.ep_base[p.ep_rank] + p.ep_off_ctr);
    int ok = 1;
    const unsigned* cw = ctr + (par ^ 1);
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(cw) : "memory");
    if (v < (unsigned)p.ep_P) {
      const unsigned long long t0 = globaltimer_ns();
      do {
        __nanosleep(64);
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(cw) : "memory");
        if (globaltimer_ns() - t0 > 20000000000ull) {
          atomicExch(ctr + 4, 1u);
          ok = 0;
          break;
        }
      } while (v < (unsigned)p.ep_P);
    }
    if (ok) {
      ctr[par] = 0u;
      ctr[2 + par] = 0u;
    }
    s_ok = ok;
  }
  __syncthreads();
  if (s_ok && p.ep_shared_dev) pdl_trigger();  // the grid's other CTAs have exited
}

// Shared tail of both route kernels: arrive on the token group's counter; the group's last
// CTA runs phase 2 (top-k a2, histogram + token lists a3) for its tokens; the last phase-2
// CTA of the grid flips the count parity (all CTAs have read it by then).
template <int EPL>
__device__ __forceinline__ void route_tail(const RouteParams& p, int* cnt, int par, int n0, int n1,
                                           unsigned long long* tr, int& s_flag) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int E = p.E;
  __syncthreads();
  if (tid == 0) {
    if (tr) tr[1] = globaltimer_ns();
    // release this CTA's logits; acquire the earlier arrivals' for the group's phase 2.
    // EP: the release is at system scope, so this CTA's own peer stores (X slices) are
    // published by the CTA itself (after the barrier, cumulative over its threads), not
    // only through the gpu-scope arrival chain to the grid's last CTA
    const int old = p.ep_P > 1 ? atom_add_acq_rel_sys(&p.g_cnt[blockIdx.y], 1)
                           : atom_add_acq_rel_gpu(&p.g_cnt[blockIdx.y], 1);
    s_flag = old == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (!s_flag) return;
  if (tid == 0) {
    p.g_cnt[blockIdx.y] = 0;
    if (tr) tr[2] = globaltimer_ns();
  }

  // ================= phase 2: top-k of this token group (a2) + histogram (a3)
  // Lane l holds logits e = l + 32 i (i < EPL), sorts them by (value desc, id asc) in
  // registers, then k rounds of a warp argmax over the lanes' heads; the winner pops.
  for (int n = n0 + warp; n < n1; n += kRouteThreads / 32) {
    float v[EPL];
    if (p.ksplit > 1) {  // sum the fp64 slices in slice order, round once (R-17)
      double s[EPL];
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        const int e = lane + 32 * i;
        s[i] = e < E ? __ldcg(p.logits64 + (size_t)n * E + e) : 0.0;
      }
      for (int q = 1; q < p.ksplit; ++q)
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          const int e = lane + 32 * i;
          if (e < E) s[i] += __ldcg(p.logits64 + ((size_t)q * p.maxN + n) * E + e);
        }
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        const int e = lane + 32 * i;
        v[i] = e < E ? (float)s[i] : -INFINITY;
        if (e < E) p.logits[(size_t)n * E + e] = v[i];  // the fp32 logits (debug output)
      }
    } else {
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        const int e = lane + 32 * i;
        v[i] = e < E ? __ldcg(p.logits + (size_t)n * E + e) : -INFINITY;
      }
    }
    if (tr && n == n0) {  // debug: logits arrived (in-order issue after a use of every value)
      float s = 0.f;
#pragma unroll
      for (int i = 0; i < EPL; ++i) s += v[i];
      if (s == 1.2345e-30f) tr[7] = 1;
      if (lane == 0) tr[4] = globaltimer_ns();
    }
    route_token<EPL>(p, cnt, par, n, v, (tr && n == n0) ? tr : nullptr);
  }
  if (tr && tid == 0) tr[6] = globaltimer_ns();
  __syncthreads();
  if (tid == 0) {
    if (tr) tr[3] = globaltimer_ns();
    // every CTA has read par; EP: system-scope release of this CTA's peer top-k / gate stores
    const int old = p.ep_P > 1 ? atom_add_acq_rel_sys(p.g_done, 1) : atom_add_acq_rel_gpu(p.g_done, 1);
    s_flag = old == (int)gridDim.y - 1;  // the grid's last CTA
    if (old == (int)gridDim.y - 1) {
      *p.g_done = 0;
      *p.par = par ^ 1;  // consumers (FFN, book) read this step's counts at cnt2[par ^ 1]
      if (p.ep_P > 1) {  // every CTA's peer stores precede this point (each CTA released
                         // them itself; the g_cnt / g_done chains acquired them here): one
                         // system-scope release fence, then the arrivals.  World 1 has no
                         // peer: the FFN's wait on this grid orders everything (stream order)
        fence_release_sys();
        for (int dst = 0; dst < p.ep_P; ++dst)
          red_relaxed_sys_add_u32(reinterpret_cast<unsigned*>(p.ep_base[dst] + p.ep_off_ctr) + (par ^ 1), 1u);
      }
    }
  }
  if (p.ep_lists && p.ep_P > 1) route_ep_wait(p, par, s_flag);
}

// Peer-memory EP dispatch of X: CTA (bx, by) stores uint4 columns [bx*per, (bx+1)*per) of
// its token rows [n0, n1) into every rank's x_all (the grid's CTAs share each row).
template <typename T>
__device__ __forceinline__ void route_ep_push_x(const RouteParams& p, int n0, int n1) {
  if (!p.ep_P) return;
  const int u4 = p.H * (int)sizeof(T) / 16;
  const int per = (u4 + (int)gridDim.x - 1) / (int)gridDim.x;
  const int q0 = blockIdx.x * per, w = min(u4, q0 + per) - q0, rows = n1 - n0;
  if (w <= 0 || rows <= 0) return;
  const int tot = p.ep_P * rows * w;
  for (int i = threadIdx.x; i < tot; i += blockDim.x) {
    const int q = q0 + i % w, n = n0 + (i / w) % rows, dst = i / (w * rows);
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(static_cast<const T*>(p.x) + (size_t)n * p.H) + q);
    reinterpret_cast<uint4*>(p.ep_base[dst] + p.ep_off_x)[((size_t)p.ep_rank * p.maxN + n) * u4 + q] = v;
  }
}

// grid (ceil(E/8), ceil(N/tpc)), 256 threads.  EPL = logits per lane in the top-k
// (power of two >= E/32).
template <typename T, int EPL>
__global__ void __launch_bounds__(kRouteThreads) tide_route_kernel(const __grid_constant__ RouteParams p) {
  __shared__ int s_flag;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int E = p.E, N = p.N, H = p.H;
  const int n0 = blockIdx.y * p.tpc, n1 = min(N, n0 + p.tpc);
  pdl_wait();     // X may be written by the previous kernel in the stream
  // let the FFN grid start its prologue; peer-memory EP with a peer on this GPU: only once the
  // local lists exist (route_ep_lists), so a resident FFN never holds SMs that peer still needs
  if (!p.ep_lists || !p.ep_shared_dev) pdl_trigger();
  unsigned long long* tr =
      p.trace ? p.trace + 8 * ((size_t)blockIdx.y * gridDim.x + blockIdx.x) : nullptr;
  if (tr && tid == 0) { tr[0] = globaltimer_ns(); tr[1] = tr[2] = tr[3] = tr[4] = tr[5] = tr[6] = 0; }
  const int par = __ldcg(p.par);  // read before this CTA arrives: the flip comes after all arrive
  int* cnt = p.cnt2 + par * E;
  if (blockIdx.x == 0 && blockIdx.y == 0) {
    for (int i = tid; i < E; i += blockDim.x) p.cnt2[(par ^ 1) * E + i] = 0;
    for (int i = tid; i < p.n_zero; i += blockDim.x) p.zero_i[i] = 0;
    if (p.ep_P) {  // the next step's half of this rank's local-expert counts (see route_token)
      int* c2 = reinterpret_cast<int*>(p.ep_base[p.ep_rank] + p.ep_off_cnt) + (par ^ 1) * p.ep_El;
      for (int i = tid; i < p.ep_El; i += blockDim.x) c2[i] = 0;
    }
  }

  // ================= phase 1: router logits (a1)
  {
    constexpr int G = 8;  // 16-byte chunks in flight per lane per group
    const int e = blockIdx.x * kRouterWarps + warp;
    const int chunks = H * (int)sizeof(T) / 16;
    const bool copy_x = blockIdx.x == 0 && warp == 0 && !p.ep_P;  // EP: x_all (push_x)
    if (e < E) {
      const uint4* wrow = reinterpret_cast<const uint4*>(static_cast<const T*>(p.wr) + (size_t)e * H);
      for (int n = n0; n < n1; n += 2) {
        const bool two = n + 1 < n1;
        const uint4* x0 = reinterpret_cast<const uint4*>(static_cast<const T*>(p.x) + (size_t)n * H);
        const uint4* x1 = reinterpret_cast<const uint4*>(static_cast<const T*>(p.x) + (size_t)(two ? n + 1 : n) * H);
        uint4* y0 = reinterpret_cast<uint4*>(static_cast<T*>(p.x_in) + (size_t)n * H);
        uint4* y1 = reinterpret_cast<uint4*>(static_cast<T*>(p.x_in) + (size_t)(two ? n + 1 : n) * H);
        double a0 = 0.0, a1 = 0.0;
        for (int base = 0; base < chunks; base += 32 * G) {
          uint4 wv[G], xv0[G], xv1[G];
#pragma unroll
          for (int i = 0; i < G; ++i) {
            const int c = base + lane + 32 * i;
            if (c < chunks) {
              wv[i] = __ldg(wrow + c);
              xv0[i] = __ldg(x0 + c);
              xv1[i] = __ldg(x1 + c);
            }
          }
#pragma unroll
          for (int i = 0; i < G; ++i) {
            const int c = base + lane + 32 * i;
            if (c < chunks) {
              a0 += (double)chunk_dot<T>(xv0[i], wv[i]);
              a1 += (double)chunk_dot<T>(xv1[i], wv[i]);
              if (copy_x) {
                y0[c] = xv0[i];
                y1[c] = xv1[i];
              }
            }
          }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          a0 += __shfl_xor_sync(0xffffffffu, a0, o);
          a1 += __shfl_xor_sync(0xffffffffu, a1, o);
        }
        if (lane == 0) {
          p.logits[(size_t)n * E + e] = (float)a0;
          if (two) p.logits[(size_t)(n + 1) * E + e] = (float)a1;
        }
      }
    }
  }
  route_ep_push_x<T>(p, n0, n1);
  route_tail<EPL>(p, cnt, par, n0, n1, tr, s_flag);
}

// bf16 variant, phase 1 on the tensor cores: CTA = 16 experts x 8 tokens, the 8 warps
// split H; each warp issues m16n8k16 MMAs with C = 0 and adds every 16-product partial into
// fp64 registers, then the 8 warp partials are summed in warp order in fp64 and rounded
// to fp32 once (R-17: the only fp32 roundings are inside each 16-term MMA sum).
// k is permuted identically in A and B: lane (g, c) loads 16 contiguous bytes at
// k = kb + 8c of expert rows g, g+8 and token g; its bf16 pairs 0,1 feed k-slots
// {2c, 2c+8} of the first MMA, pairs 2,3 those of the second, so the two MMAs cover
// exactly k in [kb, kb+32).  grid (E/16, ceil(N/8)), 256 threads; needs E % 16 == 0,
// H % 256 == 0.
// G = 32-wide k blocks in flight per warp per round (8: one load round at H=2048);
// MINB = resident CTAs per SM the register budget is sized for.  (G=4 with 4 CTAs/SM was
// measured for the 512-CTA sweep grid: one wave, but no faster end to end.)
template <int EPL, int G, int MINB>
__global__ void __launch_bounds__(kRouteThreads, MINB) tide_route_tc_kernel(const __grid_constant__ RouteParams p) {
  __shared__ int s_flag;
  __shared__ double s_red[kRouteThreads / 32][32][4];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int E = p.E, N = p.N, H = p.H;
  const int S = p.ksplit, ks = blockIdx.x % S;  // this CTA's slice of H (S slices per tile)
  const int n0 = blockIdx.y * 8, n1 = min(N, n0 + 8), e0 = (blockIdx.x / S) * 16;
  pdl_wait();
  if (!p.ep_lists || !p.ep_shared_dev) pdl_trigger();  // see tide_route_kernel
  unsigned long long* tr =
      p.trace ? p.trace + 8 * ((size_t)blockIdx.y * gridDim.x + blockIdx.x) : nullptr;
  if (tr && tid == 0) { tr[0] = globaltimer_ns(); tr[1] = tr[2] = tr[3] = tr[4] = tr[5] = tr[6] = 0; }
  const int par = __ldcg(p.par);
  int* cnt = p.cnt2 + par * E;
  if (blockIdx.x == 0 && blockIdx.y == 0) {
    for (int i = tid; i < E; i += blockDim.x) p.cnt2[(par ^ 1) * E + i] = 0;
    for (int i = tid; i < p.n_zero; i += blockDim.x) p.zero_i[i] = 0;
    if (p.ep_P) {  // the next step's half of this rank's local-expert counts (see route_token)
      int* c2 = reinterpret_cast<int*>(p.ep_base[p.ep_rank] + p.ep_off_cnt) + (par ^ 1) * p.ep_El;
      for (int i = tid; i < p.ep_El; i += blockDim.x) c2[i] = 0;
    }
  }
  // ================= phase 1: router logits (a1)
  {
    const int g = lane >> 2, c = lane & 3;
    const __nv_bfloat16* wr = static_cast<const __nv_bfloat16*>(p.wr);
    const uint4* wa = reinterpret_cast<const uint4*>(wr + (size_t)(e0 + g) * H);
    const uint4* wb = reinterpret_cast<const uint4*>(wr + (size_t)(e0 + g + 8) * H);
    const uint4* xt = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(p.x) +
                                                     (size_t)max(0, min(n0 + g, N - 1)) * H);
    // this warp's k range: slice ks of H, split over the 8 warps
    const int kw = H / (S * (kRouteThreads / 32)), kbeg = ks * (H / S) + warp * kw;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int kb = kbeg; kb < kbeg + kw; kb += 32 * G) {
      uint4 A0[G], A1[G], B[G];
#pragma unroll
      for (int i = 0; i < G; ++i) {
        const int k = kb + 32 * i;
        if (k < kbeg + kw) {
          const int q = (k >> 3) + c;  // uint4 index of k + 8c
          A0[i] = __ldg(wa + q);
          A1[i] = __ldg(wb + q);
          B[i] = __ldg(xt + q);
        }
      }
#pragma unroll
      for (int i = 0; i < G; ++i) {
        if (kb + 32 * i < kbeg + kw) {
          float d[4];
          mma_bf16_m16n8k16(d, A0[i].x, A1[i].x, A0[i].y, A1[i].y, B[i].x, B[i].y);
#pragma unroll
          for (int r = 0; r < 4; ++r) acc[r] += (double)d[r];
          mma_bf16_m16n8k16(d, A0[i].z, A1[i].z, A0[i].w, A1[i].w, B[i].z, B[i].w);
#pragma unroll
          for (int r = 0; r < 4; ++r) acc[r] += (double)d[r];
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) s_red[warp][lane][r] = acc[r];
    // x_in copy (the FFN's gather source), spread over the token group's expert tiles: CTA bx
    // copies uint4 columns [bx*per, (bx+1)*per) of the group's rows (no straggler CTA); under
    // EP the FFN gathers from x_all instead (route_ep_push_x)
    if (!p.ep_P) {
      const int per_row = H / 8;  // uint4 per row
      const int per = (per_row + (int)gridDim.x - 1) / (int)gridDim.x;
      const int q0 = blockIdx.x * per, w = min(per_row, q0 + per) - q0;
      for (int i = tid; i < (n1 - n0) * w; i += blockDim.x) {
        const int n = n0 + i / w, q = q0 + i % w;
        reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.x_in) + (size_t)n * H)[q] =
            __ldg(reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(p.x) + (size_t)n * H) + q);
      }
    }
    __syncthreads();
    if (tid < 128) {  // output (expert row r, token col q): lane (r&7)*4 + q/2, reg 2(r>>3) + (q&1)
      const int r = tid >> 3, q = tid & 7;
      const int ln = (r & 7) * 4 + (q >> 1), rg = (r >> 3) * 2 + (q & 1);
      double v = 0.0;
#pragma unroll
      for (int w = 0; w < kRouteThreads / 32; ++w) v += s_red[w][ln][rg];
      if (n0 + q < N) {
        if (S == 1)
          p.logits[(size_t)(n0 + q) * E + e0 + r] = (float)v;
        else  // fp64 partial of this K slice; phase 2 sums the S slices in order
          p.logits64[((size_t)ks * p.maxN + n0 + q) * E + e0 + r] = v;
      }
    }
  }
  route_ep_push_x<__nv_bfloat16>(p, n0, n1);
  route_tail<EPL>(p, cnt, par, n0, n1, tr, s_flag);
}

// One CTA (1024 threads): a4 placement and a5 bookkeeping from the hit counts.
// dynamic smem: 6 * E ints.
__global__ void __launch_bounds__(1024) tide_book_kernel(const __grid_constant__ BookParams p) {
  extern __shared__ int book_smem[];
  __shared__ int s_scratch[33];
  __shared__ int s_cnt, s_prom, s_evic, s_rp, s_uq;
  const int tid = threadIdx.x;
  const int E = p.E, N = p.N, k = p.k;
  const int NW = (N + 31) >> 5;
  int* s_hits = book_smem;
  int* s_pl = s_hits + E;
  int* s_order = s_pl + E;
  int* s_bstart = s_order + E;
  int* s_tmp = s_bstart + E;
  int* s_key = s_tmp + E;  // the counts that rank experts at this step (NEXT-1)
  if (tid == 0) { s_cnt = 0; s_prom = 0; s_evic = 0; s_rp = 0; s_uq = 0; }
  const int* cnt = p.par ? p.cnt + (__ldcg(p.par) ^ 1) * E : p.cnt;
  for (int e = tid; e < E; e += blockDim.x) {
    s_hits[e] = __ldcg(cnt + e);
    s_key[e] = (p.mode == 0 || p.step == 0) ? s_hits[e] : p.acc[e];
    s_pl[e] = p.placement_in[e] != 0;  // incumbents (overwritten below)
  }
  __syncthreads();
  if (p.pf_list) {  // NEXT-3: rank this step's hit experts for the previous layer's prefetch
    // by id (the FFN's claim order: the prefetched experts are the ones its first wave
    // streams) or by hits (pf_by_hits)
    for (int e = tid; e < E; e += blockDim.x) {
      const int he = s_hits[e];
      if (he > 0) {
        int r = 0;
        for (int f = 0; f < E; ++f) {
          const int hf = s_hits[f];
          r += p.pf_by_hits ? ((hf > he) || (hf == he && f < e)) : (hf > 0 && f < e);
        }
        p.pf_list[r] = e;  // hit experts occupy ranks 0..U-1
      }
    }
    const int u = __syncthreads_count(tid < E && s_hits[tid] > 0);  // E <= blockDim
    if (tid == 0) *p.pf_n = u;
  }
  if (p.refresh) {  // rank(e) = #{f : key[f] > key[e] or (== and [incumbent f] or f < e)}
    const int S = max(1, (int)blockDim.x / E);   // threads per expert
    const int seg = (E + S - 1) / S;
    for (int e = tid; e < E; e += blockDim.x) s_tmp[e] = 0;
    __syncthreads();
    for (int idx = tid; idx < E * S; idx += blockDim.x) {
      const int e = idx % E, sg = idx / E;
      const int f0 = sg * seg, f1 = min(E, f0 + seg);
      const int he = s_key[e];
      const int ie = p.incumbent ? s_pl[e] : 0;
      int r = 0;
#pragma unroll 8
      for (int f = f0; f < f1; ++f) {
        const int hf = s_key[f];
        const int jf = p.incumbent ? s_pl[f] : 0;
        r += (hf > he) || (hf == he && (jf > ie || (jf == ie && f < e)));
      }
      atomicAdd(&s_tmp[e], r);
    }
    __syncthreads();
    for (int e = tid; e < E; e += blockDim.x) s_pl[e] = s_tmp[e] < p.capacity;
  } else {
    for (int e = tid; e < E; e += blockDim.x)
      if (s_pl[e]) atomicAdd(&s_cnt, 1);
  }
  __syncthreads();
  int* info_hits = reinterpret_cast<int*>(p.info + 1);
  uint8_t* info_pl = reinterpret_cast<uint8_t*>(info_hits + E);
  for (int e = tid; e < E; e += blockDim.x) {
    p.hit_counts[e] = s_hits[e];
    info_hits[e] = s_hits[e];
  }
  if (!p.refresh && s_cnt > p.capacity) {  // S:49, S:263 budget safety
    for (int e = tid; e < E; e += blockDim.x) {  // placement' = the (unchanged) input
      p.placement_out[e] = (uint8_t)s_pl[e];
      info_pl[e] = (uint8_t)s_pl[e];
    }
    for (int i = tid; i < E * NW; i += blockDim.x) p.mask_rw[i] = 0u;
    if (tid == 0) p.info->status = 3;
    return;
  }
  if (p.mode != 0)  // NEXT-1 counter state after this step
    for (int e = tid; e < E; e += blockDim.x)
      p.acc[e] = ((p.step == 0 || (p.mode == 1 && p.refresh)) ? 0 : p.acc[e]) + s_hits[e];
  for (int e = tid; e < E; e += blockDim.x) {
    const int was = p.placement_in[e] != 0, res = s_pl[e];
    if (res && !was) atomicAdd(&s_prom, 1);
    if (was && !res) atomicAdd(&s_evic, 1);
    if (res) atomicAdd(&s_rp, s_hits[e]);
    if (s_hits[e] > 0) atomicAdd(&s_uq, 1);
    p.placement_out[e] = (uint8_t)res;
    info_pl[e] = (uint8_t)res;
    s_tmp[e] = res;
  }
  __syncthreads();
  // bucket order: resident ascending id, then non-resident ascending id (R-11)
  const int n_res = block_scan_excl(s_tmp, E, s_scratch);
  for (int e = tid; e < E; e += blockDim.x) {
    const int rb = s_tmp[e];
    s_order[s_pl[e] ? rb : n_res + (e - rb)] = e;
  }
  __syncthreads();
  for (int i = tid; i < E; i += blockDim.x) s_tmp[i] = s_hits[s_order[i]];
  __syncthreads();
  block_scan_excl(s_tmp, E, s_scratch);  // offsets over bucket positions
  for (int i = tid; i < E; i += blockDim.x) {
    s_bstart[s_order[i]] = s_tmp[i];
    p.order[i] = s_order[i];
    p.offsets[i] = s_tmp[i];
  }
  if (tid == 0) p.offsets[E] = N * k;
  __syncthreads();
  // pos[n,j] = bucket start of its expert + lower tokens that chose the same expert
  for (int q = tid; q < N * k; q += blockDim.x) {
    const int n = q / k;
    const int e = __ldcg(p.topk_idx + q);
    const unsigned* mk = p.mask + e * NW;
    int before = 0;
    for (int w = 0; w < (n >> 5); ++w) before += __popc(__ldcg(mk + w));
    before += __popc(__ldcg(mk + (n >> 5)) & ((1u << (n & 31)) - 1u));
    p.pos[q] = s_bstart[e] + before;
  }
  __syncthreads();
  for (int i = tid; i < E * NW; i += blockDim.x) p.mask_rw[i] = 0u;
  if (tid == 0) {
    p.info->status = 0;
    p.info->refreshed = p.refresh;
    p.info->promotions = s_prom;
    p.info->evictions = s_evic;
    p.info->resident_pairs = s_rp;
    p.info->unique_experts = s_uq;
  }
}

// ---------------------------------------------------------------- a10 combine
// grid (N, ceil(H / 512)), 128 threads x 4 columns.  row(n,j) = off[e] + slot(n,j), with
// off[e] = the counts of the experts before e in id order (the FFN's row rule).
// fp32 FMA over j in slot order (then the shared expert), one rounding (R-14).
template <typename T>
__global__ void __launch_bounds__(128) tide_combine_kernel(const float* __restrict__ y,
                                                           const float* __restrict__ gates,
                                                           const int* __restrict__ topk,
                                                           const int* __restrict__ pair_slot,
                                                           const int* __restrict__ cnt2,
                                                           const int* __restrict__ par, int E,
                                                           T* __restrict__ out, int N, int k,
                                                           int H, int shared,
                                                           unsigned long long* trace) {
  extern __shared__ int s_off[];  // [E] (dynamic: the CTA must fit beside a resident FFN CTA)
  __shared__ int s_scratch[33];
  const int n = blockIdx.x, lane = threadIdx.x & 31;
  const int c = (blockIdx.y * blockDim.x + threadIdx.x) * 4;
  // Everything from the route kernel is read before the wait: it completed before the FFN
  // (the preceding grid) triggered this launch.  Lane j < k fetches pair j's expert, slot and
  // gate; the CTA scans the per-expert counts into the row offsets off[] (one L2 round trip
  // and a CTA scan that overlap the FFN's tail).  Only y comes from the FFN, after the wait.
  int e_j = 0, s_j = 0, r_j = 0;
  float g_j = 0.f;
  if (lane < k) {
    const int q = n * k + lane;
    e_j = __ldcg(topk + q);
    s_j = __ldcg(pair_slot + q);
    g_j = __ldcg(gates + q);
  }
  {
    const int* cnt = cnt2 + (__ldcg(par) ^ 1) * E;  // this step's half (route.cuh RouteParams)
    for (int e = threadIdx.x; e < E; e += blockDim.x) s_off[e] = __ldcg(cnt + e);
    __syncthreads();
    block_scan_excl(s_off, E, s_scratch);
  }
  pdl_wait();
  pdl_trigger();
  if (trace && threadIdx.x == 0) atomicMax(trace, globaltimer_ns());  // debug: latest start
  if (lane < k) r_j = s_off[e_j] + s_j;
  const bool valid = c < H;  // (lanes stay converged for the shuffles)
  const int cc = valid ? c : 0;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 8
  for (int j = 0; j < k; ++j) {
    const int r = __shfl_sync(0xffffffffu, r_j, j);
    const float g = __shfl_sync(0xffffffffu, g_j, j);
    const float4 v = __ldcg(reinterpret_cast<const float4*>(y + (size_t)r * H + cc));
    acc.x = fmaf(g, v.x, acc.x);
    acc.y = fmaf(g, v.y, acc.y);
    acc.z = fmaf(g, v.z, acc.z);
    acc.w = fmaf(g, v.w, acc.w);
  }
  if (!valid) return;
  if (shared) {
    const float4 v = __ldcg(reinterpret_cast<const float4*>(y + (size_t)(N * k + n) * H + c));
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
  if (trace && threadIdx.x == 0) atomicMax(trace + 1, globaltimer_ns());  // debug: latest end
}

}  // namespace tide
