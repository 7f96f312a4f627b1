// tide.cu -- host runtime + C ABI (include/tide.h) of the TIDE MoE layer-step.
//
// One tide_ctx per (layer, device).  It owns the workspaces, the HBM slot pool
// (capacity experts) and staging ring for host_master mode, a side stream, events
// and cached TMA tensor maps.  A step is, on the caller's stream:
//
//   tide_route_kernel    a1 router, a2 top-k/gates, a3 hits + per-expert token lists
//   tide_ffn_kernel      a7/a9 grouped SwiGLU over the hit experts already in HBM (+ shared)
//   [host_master only: read the bookkeeping info, enqueue H2D copies of the missing
//    experts on the side stream (a6), tide_ffn_kernel per staged chunk once its copy
//    event fires (a8)]
//   tide_combine_kernel  a10
//
// and, concurrently on the side stream (device_all) or before the FFN (host_master),
//   tide_book_kernel     a4 refresh/placement, a5 bucket order/offsets/pos, info block.
// Consecutive kernels on the caller's stream use programmatic dependent launch.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include <nccl.h>

#include "../../include/tide.h"
#include "analytics.cuh"
#include "ep.cuh"
#include "ffn.cuh"
#include "route.cuh"

using namespace tide;

namespace {

thread_local std::string g_err;

tide_status fail(tide_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

#define NC_TRY(expr)                                                                     \
  do {                                                                                   \
    ncclResult_t r_ = (expr);                                                            \
    if (r_ != ncclSuccess)                                                               \
      return fail(TIDE_ENCCL, "%s failed: %s (%s:%d)", #expr, ncclGetErrorString(r_),     \
                  __FILE__, __LINE__);                                                   \
  } while (0)

#define CU_TRY(expr)                                                                     \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(TIDE_ECUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_),     \
                  __FILE__, __LINE__);                                                   \
  } while (0)

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2-D map over a row-major [rows, cols] matrix; box = (128 B of columns) x box_rows,
// 128-byte swizzle (matches smem_desc_sw128).
tide_status make_map(CUtensorMap* m, const void* base, bool bf16, uint64_t cols, uint64_t rows,
                     uint32_t box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(TIDE_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const uint32_t eb = bf16 ? 2 : 4;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * eb};
  cuuint32_t box[2] = {128u / eb, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                  const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(TIDE_ECUDA, "cuTensorMapEncodeTiled failed (%d) cols=%llu rows=%llu", (int)r,
                (unsigned long long)cols, (unsigned long long)rows);
  return TIDE_OK;
}

}  // namespace

struct tide_ctx {
  tide_layer_desc d;
  int capacity = 0, staging = 0, device = 0, num_sms = 148;
  int E = 0, k = 0, H = 0, F = 0, maxN = 0, NWmax = 1;
  bool bf16 = true;
  size_t eb = 2, expert_elems = 0, expert_bytes = 0;
  int max_rows = 0, max_entries = 0;
  int ffn_smem = 0;  // the FFN's dynamic smem: ring + barriers + a work list of max_entries

  // workspaces (device)
  float* logits = nullptr;
  int* topk = nullptr;
  float* gates = nullptr;
  int* pair_slot = nullptr;
  int* cnt = nullptr;        // [2][E] per-expert token counts (double-buffered, see cnt_par)
  int* cnt_par = nullptr;    // [2] device parity word + route completion counter
  // NEXT-3 cross-layer prefetch
  int* pf_list = nullptr;    // [E] this layer's hit experts ranked by hits (written by book)
  int* pf_n = nullptr;       // [1] their number
  bool pf_target = false;    // some other context prefetches for this one: book ranks
  tide_ctx* pf_next = nullptr;         // the layer this context prefetches for
  const void* pf_weights = nullptr;    // its packed experts (device_all)
  int pf_max = 0;                      // budget in experts
  int64_t pf_budget = 0;               // budget in bytes
  // NEXT-3 H2D prefetch (host_master mode)
  tide_ctx* pf_next_h = nullptr;       // the layer this context prefetches host experts for
  int pf_slots_req = 0;                // prefetch slots of this context (set before its pool)
  std::vector<int> pf_exp;             // expert in each prefetch slot (-1 free)
  std::vector<cudaEvent_t> pf_ev;      // its H2D copy done
  cudaEvent_t ev_pf_free = nullptr;    // this context's last step is done with the slots
  std::vector<int> last_streamed;      // experts streamed at the last step, most-hit first
  const void* last_master = nullptr;   // the host master of the last step
  int pf_issued = 0;                   // H2D copies issued for this context's next step
  int pf_min_hits = 2;                 // predict experts streamed with >= this many hits
                                       // (TIDE_H2D_PF_MIN_HITS)
  int* list = nullptr;       // [E * maxN] per-expert token lists
  unsigned* mask = nullptr;  // [E * NWmax] per-expert token bitmasks
  int* g_cnt = nullptr;      // [maxN + 2] route-kernel last-CTA counters
  int* off = nullptr;        // [E] FFN row offset of each expert (id order)
  int* pos = nullptr;
  int* order = nullptr;
  int* offsets = nullptr;
  void* x_in = nullptr;      // [maxN, H] copy of the block's hidden states (gather4 source)
  void* h_perm = nullptr;    // [max_rows, F]
  float* y_perm = nullptr;   // [max_rows, H]
  // A/B measurement knobs, read once from the environment at context creation:
  // TIDE_ROUTE_TPC (tokens per CUDA-core router CTA), TIDE_ROUTER_CC=1 (CUDA-core router for
  // bf16), TIDE_ROUTE_ONE_PER_SM=1 (one router CTA per SM), (see DESIGN 11
  // for the measured negative results that removed other knobs)
  int knob_route_tpc = 0;
  bool knob_router_cc = false, knob_route_one_per_sm = false;
  bool knob_route_ksplit1 = false;  // TIDE_ROUTE_KSPLIT1=1: one router CTA per 16 x 8 tile
  bool knob_pf_by_hits = false;    // TIDE_PF_BY_HITS=1: prefetch ranked by hits, no shared expert
  bool knob_pf_whole = false;      // TIDE_PF_WHOLE_EXPERT=1: prefetch whole experts (not gate/up)
  int64_t pf_self_bytes = -1;      // own-layer prefetch before the FFN's routing wait (-1: half
                                   // the previous layer's tail budget; TIDE_PF_SELF_MB overrides)
  int64_t pf_prev_budget = 0;      // budget of the context whose FFN tail prefetches this layer
  double* logits64 = nullptr;       // [2][maxN][E] fp64 router partials (bf16, TC router)
  int* ffn_ctrl = nullptr;   // [2 + max_entries]: scheduler counter, per-entry done counters,
                             // grid arrival counter (peer-memory EP)
  RouteInfo* info = nullptr; // + hits[E] + placement[E]
  size_t info_bytes = 0;
  int* slot_of_dev = nullptr;
  int* counter_acc = nullptr;  // [E] NEXT-1 counter state

  // host_master mode
  void* pool = nullptr;            // (capacity + staging) packed experts
  int4* entries2 = nullptr;        // staged-chunk work lists (device)
  int* ctrl2 = nullptr;            // per chunk {n_entries, sched}
  int* done2 = nullptr;
  int max_chunks = 0, max_entries2 = 0;
  void* h_info = nullptr;          // pinned mirror of the info block
  int4* h_entries2 = nullptr;      // pinned
  int* h_ctrl2 = nullptr;          // pinned (ctrl2 + done2 zeros)
  int* h_slot_of = nullptr;        // pinned mirror of slot_of_dev
  std::vector<int> slot_of;        // expert -> pool slot (authoritative)
  std::vector<int> owner;          // pool slot -> expert (-1 free)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_route = nullptr, ev_book = nullptr, ev_info = nullptr, ev_gemm1 = nullptr,
              ev_side_done = nullptr;
  std::vector<cudaEvent_t> ev_chunk_ready, ev_chunk_done;

  // cached tensor maps
  CUtensorMap map_x, map_h, map_gu, map_d, map_gu_s, map_d_s;
  const void* map_src = nullptr;
  int map_src_rows = 0;
  const void* map_shared_src = nullptr;
  bool have_shared_map = false;

  // expert parallelism (tide_ctx_create_ep)
  bool ep = false;
  int rank = 0, world = 1, El = 0, e0 = 0, rows_all = 0;
  ncclComm_t comm = nullptr;
  bool own_comm = false;
  void* x_all = nullptr;        // [P*maxN, H] all ranks' tokens
  int* topk_all = nullptr;      // [P*maxN, k]
  float* gates_all = nullptr;   // [P*maxN, k]
  int* pslot_all = nullptr;     // [P*maxN, k]
  int* cnt_l = nullptr;         // [El] local experts' token counts over all rows
  int* list_l = nullptr;        // [El, P*maxN]
  int* off_l = nullptr;         // [El]
  int* hits_l = nullptr;        // [El] scratch
  float* partial = nullptr;     // [P*maxN, H] per-source partial sums (send buffer)
  float* recv = nullptr;        // [P*maxN, H] partials for this rank's tokens
  CUtensorMap map_x_all;
  // peer-memory EP (tide_ctx_create_ep_p2p): x_all/topk_all/gates_all/recv live in `sym`
  bool p2p = false, connected = false;
  bool peer_same_device = false;  // a peer's symmetric region lives on this GPU (R-22)
  char* sym = nullptr;
  EpSymLayout lay{};
  EpPeers peers{};
  std::vector<void*> ipc_opened;  // peers' regions opened with cudaIpcOpenMemHandle
  cudaEvent_t ev_ep_done = nullptr;  // the last EP step's completion (tide_ctx_ep_wait)
  unsigned* dst_l = nullptr;      // [El, rows_all] owner rank << 28 | pair row of each list slot (p2p)
  int ep_arrivals = 0;            // p2p: combine arrivals per step = sum of the ranks' FFN grids

  // per-phase timing (tide_ctx_set_timing)
  bool timing = false;
  struct Rec { cudaEvent_t ev[7]; int64_t launches, ffn_launches; };
  std::vector<cudaEvent_t> ev_pool;
  std::vector<Rec> pending;
  tide_phase_times acc{};
  int64_t launches = 0, ffn_launches = 0;  // kernels launched by this context (lifetime)
};

static cudaEvent_t take_event(tide_ctx* c) {
  if (!c->ev_pool.empty()) {
    cudaEvent_t e = c->ev_pool.back();
    c->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

static int route_epl(int E) {
  const int need = (E + 31) / 32;
  int epl = 1;
  while (epl < need) epl <<= 1;
  return epl;
}

// Load every kernel a peer-memory EP step launches now.  With lazy module loading the
// first launch of a kernel can synchronise the device; a rank whose kernels spin on a peer
// must never block on that between its own launches (CUDA_MODULE_LOADING=LAZY hazard for
// producer/consumer kernels).
template <typename F>
static void touch(F* f) {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, f);
}
static void preload_ep_p2p_kernels(const tide_ctx* c) {
  const int epl = route_epl(c->E);
  if (c->bf16 && c->E % 16 == 0 && c->H % 256 == 0) {
    // both register budgets: launch_route picks MINB = 2 when the grid exceeds one wave
#define TOUCH_TC(EP) \
  do { touch(tide_route_tc_kernel<EP, 8, 1>); touch(tide_route_tc_kernel<EP, 8, 2>); } while (0)
    switch (epl) {
      case 1: TOUCH_TC(1); break;
      case 2: TOUCH_TC(2); break;
      case 4: TOUCH_TC(4); break;
      case 8: TOUCH_TC(8); break;
      case 16: TOUCH_TC(16); break;
      default: TOUCH_TC(32); break;
    }
#undef TOUCH_TC
  }
#define TOUCH_ROUTE(TT)                                     \
  switch (epl) {                                            \
    case 1: touch(tide_route_kernel<TT, 1>); break;         \
    case 2: touch(tide_route_kernel<TT, 2>); break;         \
    case 4: touch(tide_route_kernel<TT, 4>); break;         \
    case 8: touch(tide_route_kernel<TT, 8>); break;         \
    case 16: touch(tide_route_kernel<TT, 16>); break;       \
    default: touch(tide_route_kernel<TT, 32>); break;       \
  }
  touch(tide_book_kernel);  // the side-stream placement kernel of the EP step
  if (c->bf16) {
    TOUCH_ROUTE(__nv_bfloat16)
    touch(tide_ffn_kernel<__nv_bfloat16, true>);
    touch(tide_ep_final_p2p_kernel<__nv_bfloat16>);
  } else {
    TOUCH_ROUTE(float)
    touch(tide_ffn_kernel<float, true>);
    touch(tide_ep_final_p2p_kernel<float>);
  }
#undef TOUCH_ROUTE
  touch(tide_book_kernel);
}

extern "C" {

int32_t tide_abi_version(void) { return TIDE_ABI_VERSION; }
int32_t tide_build_sm(void) { return 100; }
const char* tide_last_error(void) { return g_err.c_str(); }

size_t tide_expert_elems(const tide_layer_desc* d) {
  return d ? (size_t)3 * d->hidden * d->ffn : 0;
}
size_t tide_expert_bytes(const tide_layer_desc* d) {
  return d ? tide_expert_elems(d) * (d->dtype == TIDE_BF16 ? 2 : 4) : 0;
}

tide_status tide_pack_expert(const tide_layer_desc* d, const void* wg, const void* wu,
                             const void* wd, void* dst, void* stream) {
  if (!d || !wg || !wu || !wd || !dst) return fail(TIDE_EINVAL, "tide_pack_expert: null argument");
  const size_t mb = (size_t)d->hidden * d->ffn * (d->dtype == TIDE_BF16 ? 2 : 4);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint8_t* o = static_cast<uint8_t*>(dst);
  CU_TRY(cudaMemcpyAsync(o, wg, mb, cudaMemcpyDefault, s));
  CU_TRY(cudaMemcpyAsync(o + mb, wu, mb, cudaMemcpyDefault, s));
  CU_TRY(cudaMemcpyAsync(o + 2 * mb, wd, mb, cudaMemcpyDefault, s));
  return TIDE_OK;
}

static tide_status validate_desc(const tide_layer_desc* d) {
  if (!d) return fail(TIDE_EINVAL, "desc is null");
  if (d->num_experts < 1 || d->num_experts > 1024)
    return fail(TIDE_EUNSUPPORTED, "num_experts %d outside [1, 1024]", d->num_experts);
  if (d->top_k < 1 || d->top_k > d->num_experts || d->top_k > 32)
    return fail(TIDE_EINVAL, "top_k %d outside [1, min(E, 32)]", d->top_k);
  if (d->hidden < 64 || d->hidden > 16384 || d->hidden % 64)
    return fail(TIDE_EUNSUPPORTED, "hidden %d must be a multiple of 64 in [64, 16384]", d->hidden);
  if (d->ffn < 64 || d->ffn > 16384 || d->ffn % 64)
    return fail(TIDE_EUNSUPPORTED, "ffn %d must be a multiple of 64 in [64, 16384]", d->ffn);
  if (d->max_tokens < 1 || d->max_tokens > 1024)
    return fail(TIDE_EUNSUPPORTED, "max_tokens %d outside [1, 1024]", d->max_tokens);
  if (d->dtype != TIDE_BF16 && d->dtype != TIDE_F32)
    return fail(TIDE_EUNSUPPORTED, "dtype %d", (int)d->dtype);
  const int max_ent = d->num_experts + d->max_tokens * d->top_k / kMaxTok + 2 +
                      (d->max_tokens + kMaxTok - 1) / kMaxTok;
  if (max_ent > kMaxEntriesSmem)
    return fail(TIDE_EUNSUPPORTED, "E + N*k/128 too large for the FFN work list (%d > %d)",
                max_ent, kMaxEntriesSmem);
  return TIDE_OK;
}

void tide_ctx_destroy(tide_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->side) cudaStreamSynchronize(c->side);
  for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  if (c->p2p) {  // these live inside the symmetric region
    c->x_all = nullptr;
    c->cnt_l = nullptr;
    c->list_l = nullptr;
    c->dst_l = nullptr;
    cudaFree(c->sym);
  }
  void* dev[] = {c->logits, c->topk,     c->gates,   c->pair_slot, c->cnt,    c->list,
                 c->mask,   c->g_cnt,    c->off,     c->pos,       c->order,  c->offsets,
                 c->x_in,   c->h_perm,   c->y_perm,  c->ffn_ctrl,  c->info,   c->slot_of_dev,
                 c->pool,   c->entries2, c->ctrl2,   c->done2,  c->x_all,  c->topk_all,
                 c->gates_all, c->pslot_all, c->cnt_l, c->list_l, c->off_l, c->hits_l,
                 c->partial, c->recv, c->counter_acc, c->cnt_par, c->pf_list, c->pf_n,
                 c->logits64,
                 c->dst_l};
  for (void* p : dev)
    if (p) cudaFree(p);
  void* host[] = {c->h_info, c->h_entries2, c->h_ctrl2, c->h_slot_of};
  for (void* p : host)
    if (p) cudaFreeHost(p);
  for (cudaEvent_t e : c->ev_chunk_ready) cudaEventDestroy(e);
  for (cudaEvent_t e : c->ev_chunk_done) cudaEventDestroy(e);
  for (cudaEvent_t e : c->pf_ev) cudaEventDestroy(e);
  if (c->ev_pf_free) cudaEventDestroy(c->ev_pf_free);
  for (auto& r : c->pending)
    for (cudaEvent_t e : r.ev) cudaEventDestroy(e);
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  cudaEvent_t evs[] = {c->ev_route, c->ev_book, c->ev_info, c->ev_gemm1, c->ev_side_done,
                       c->ev_ep_done};
  for (cudaEvent_t e : evs)
    if (e) cudaEventDestroy(e);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->comm && c->own_comm) ncclCommDestroy(c->comm);
  delete c;
}

#define ALLOC(ptr, bytes)                                                                  \
  do {                                                                                     \
    if (cudaMalloc(reinterpret_cast<void**>(&(ptr)), (bytes)) != cudaSuccess) {           \
      tide_ctx_destroy(c);                                                                 \
      return fail(TIDE_ENOMEM, "cudaMalloc(%zu) failed for " #ptr, (size_t)(bytes));        \
    }                                                                                      \
    cudaMemset((ptr), 0, (bytes));                                                         \
  } while (0)

static tide_status ctx_create_impl(const tide_layer_desc* d, int32_t capacity,
                                   int32_t staging_slots, int32_t device, int32_t world,
                                   tide_ctx** out) {
  if (!out) return fail(TIDE_EINVAL, "out is null");
  *out = nullptr;
  tide_status s = validate_desc(d);
  if (s != TIDE_OK) return s;
  if (capacity < 1 || capacity > d->num_experts)
    return fail(TIDE_ECAPACITY, "capacity %d outside [1, %d]", capacity, d->num_experts);
  if (staging_slots < 2) return fail(TIDE_EINVAL, "staging_slots %d < 2", staging_slots);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
    return fail(TIDE_ECUDA, "no CUDA device %d", device);
  CU_TRY(cudaSetDevice(device));
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
  if (major != 10)
    return fail(TIDE_EUNSUPPORTED, "device %d is sm_%d0, this build is sm_100a", device, major);

  tide_ctx* c = new tide_ctx();
  c->d = *d;
  c->capacity = capacity;
  c->staging = staging_slots;
  c->device = device;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  c->E = d->num_experts;
  c->k = d->top_k;
  c->H = d->hidden;
  c->F = d->ffn;
  c->maxN = d->max_tokens;
  c->NWmax = (c->maxN + 31) / 32;
  c->bf16 = d->dtype == TIDE_BF16;
  c->eb = c->bf16 ? 2 : 4;
  c->expert_elems = tide_expert_elems(d);
  c->expert_bytes = tide_expert_bytes(d);
  const int E = c->E, k = c->k, N = c->maxN;
  c->world = world;
  c->rows_all = world * N;
  c->max_rows = world * N * k + N;
  c->max_entries = E / world + (world * N * k) / kMaxTok + 2 + (N + kMaxTok - 1) / kMaxTok;
  // (<= kMaxEntriesSmem: checked before the context exists.)  The FFN's smem is sized by this
  // context's work list, not the kernel's maximum: the smaller its footprint, the more room
  // for the CTAs that run beside it (book, combine)
  c->ffn_smem = kStages * kStageBytes + 2048 + 4 * kMaxTok + 16 * c->max_entries;

  ALLOC(c->logits, sizeof(float) * N * E);
  if (c->bf16) ALLOC(c->logits64, sizeof(double) * 2 * N * E);  // TC router's H-split partials
  ALLOC(c->topk, sizeof(int) * N * k);
  ALLOC(c->gates, sizeof(float) * N * k);
  ALLOC(c->pair_slot, sizeof(int) * N * k);
  ALLOC(c->cnt, sizeof(int) * 2 * E);
  ALLOC(c->cnt_par, sizeof(int) * 2);  // parity word, route completion counter
  ALLOC(c->pf_list, sizeof(int) * E);
  ALLOC(c->pf_n, sizeof(int));
  ALLOC(c->list, sizeof(int) * (size_t)E * N);
  ALLOC(c->mask, sizeof(unsigned) * E * c->NWmax);
  ALLOC(c->g_cnt, sizeof(int) * (N + 2));
  ALLOC(c->off, sizeof(int) * E);
  ALLOC(c->pos, sizeof(int) * N * k);
  ALLOC(c->order, sizeof(int) * E);
  ALLOC(c->offsets, sizeof(int) * (E + 1));
  ALLOC(c->x_in, c->eb * (size_t)N * c->H);
  ALLOC(c->h_perm, c->eb * (size_t)c->max_rows * c->F);
  ALLOC(c->y_perm, sizeof(float) * (size_t)c->max_rows * c->H);
  ALLOC(c->ffn_ctrl, sizeof(int) * (2 + c->max_entries));
  c->info_bytes = sizeof(RouteInfo) + sizeof(int) * E + E;
  ALLOC(c->info, c->info_bytes);
  ALLOC(c->slot_of_dev, sizeof(int) * E);
  ALLOC(c->counter_acc, sizeof(int) * E);
  if (cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_route, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_book, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_info, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_gemm1, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_side_done, cudaEventDisableTiming) != cudaSuccess) {
    tide_ctx_destroy(c);
    return fail(TIDE_ECUDA, "stream/event creation failed");
  }
  if (make_map(&c->map_x, c->x_in, c->bf16, c->H, N, 1) != TIDE_OK ||
      make_map(&c->map_h, c->h_perm, c->bf16, c->F, c->max_rows, 16) != TIDE_OK) {
    std::string m = g_err;
    tide_ctx_destroy(c);
    return fail(TIDE_ECUDA, "%s", m.c_str());
  }
  if (c->bf16) {
    cudaFuncSetAttribute(tide_ffn_kernel<__nv_bfloat16, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, kFfnSmemBytes);
    cudaFuncSetAttribute(tide_ffn_kernel<__nv_bfloat16, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, kFfnSmemBytes);
  } else {
    cudaFuncSetAttribute(tide_ffn_kernel<float, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kFfnSmemBytes);
    cudaFuncSetAttribute(tide_ffn_kernel<float, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kFfnSmemBytes);
  }
  cudaFuncSetAttribute(tide_book_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(sizeof(int) * 6 * E));
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    tide_ctx_destroy(c);
    return fail(TIDE_ECUDA, "ctx init: %s", cudaGetErrorString(e));
  }
  c->slot_of.assign(E, -1);
  if (const char* v = getenv("TIDE_ROUTE_TPC")) c->knob_route_tpc = std::max(1, std::min(8, atoi(v)));
  c->knob_router_cc = getenv("TIDE_ROUTER_CC") != nullptr;
  c->knob_route_one_per_sm = getenv("TIDE_ROUTE_ONE_PER_SM") != nullptr;
  c->knob_route_ksplit1 = getenv("TIDE_ROUTE_KSPLIT1") != nullptr;
  c->knob_pf_by_hits = getenv("TIDE_PF_BY_HITS") != nullptr;
  c->knob_pf_whole = getenv("TIDE_PF_WHOLE_EXPERT") != nullptr;
  if (const char* v = getenv("TIDE_PF_SELF_MB")) c->pf_self_bytes = (int64_t)(atof(v) * 1048576.0);
  if (const char* v = getenv("TIDE_H2D_PF_MIN_HITS")) c->pf_min_hits = std::max(1, atoi(v));
  *out = c;
  return TIDE_OK;
}

tide_status tide_ctx_create(const tide_layer_desc* d, int32_t capacity, int32_t staging_slots,
                            int32_t device, tide_ctx** out) {
  return ctx_create_impl(d, capacity, staging_slots, device, 1, out);
}

tide_status tide_nccl_unique_id(void* out) {
  if (!out) return fail(TIDE_EINVAL, "out is null");
  ncclUniqueId id;
  NC_TRY(ncclGetUniqueId(&id));
  memcpy(out, &id, sizeof(id));
  return TIDE_OK;
}

static tide_status ctx_create_ep_impl(const tide_layer_desc* d, int32_t device,
                                      const void* nccl_id, tide_ctx* parent, int32_t rank,
                                      int32_t world, tide_ctx** out, bool p2p = false) {
  if (!out) return fail(TIDE_EINVAL, "null argument");
  *out = nullptr;
  tide_status s = validate_desc(d);
  if (s != TIDE_OK) return s;
  if (world < 1 || rank < 0 || rank >= world) return fail(TIDE_EINVAL, "rank %d / world %d", rank, world);
  if (d->num_experts % world)
    return fail(TIDE_EUNSUPPORTED, "num_experts %d not divisible by world %d", d->num_experts, world);
  if (p2p && world > kEpMaxWorld)
    return fail(TIDE_EUNSUPPORTED, "peer-memory EP supports world <= %d", kEpMaxWorld);
  const int El = d->num_experts / world;
  const int max_ent = El + world * d->max_tokens * d->top_k / kMaxTok + 2 +
                      (d->max_tokens + kMaxTok - 1) / kMaxTok;
  if (max_ent > kMaxEntriesSmem)
    return fail(TIDE_EUNSUPPORTED, "EP work list too large (%d > %d)", max_ent, kMaxEntriesSmem);
  tide_ctx* c = nullptr;
  s = ctx_create_impl(d, d->num_experts, 2, device, world, &c);
  if (s != TIDE_OK) return s;
  c->ep = true;
  c->rank = rank;
  c->El = El;
  c->e0 = rank * El;
  const int N = c->maxN, k = c->k, R = c->rows_all;
  if (p2p) {  // one allocation holds everything the peers write (one IPC handle)
    auto up = [](size_t v) { return (v + 255) & ~(size_t)255; };
    EpSymLayout& L = c->lay;
    L.x_all = 0;
    L.cnt_l = up(L.x_all + c->eb * (size_t)R * c->H);
    L.list_l = up(L.cnt_l + sizeof(int) * 2 * (size_t)El);
    L.dst_l = up(L.list_l + sizeof(int) * (size_t)El * R);
    L.ypair = up(L.dst_l + sizeof(unsigned) * (size_t)El * R);
    L.hits_all = up(L.ypair + sizeof(float) * (size_t)N * k * c->H);
    L.ctr = up(L.hits_all + sizeof(int) * (size_t)c->E);
    L.total = up(L.ctr + sizeof(unsigned) * 8);
    c->p2p = true;
    ALLOC(c->sym, L.total);
    c->x_all = c->sym + L.x_all;
    c->cnt_l = reinterpret_cast<int*>(c->sym + L.cnt_l);  // [2][El], by step parity
    c->list_l = reinterpret_cast<int*>(c->sym + L.list_l);
    c->dst_l = reinterpret_cast<unsigned*>(c->sym + L.dst_l);
    c->peers.base[rank] = c->sym;
    {
      const unsigned g = (unsigned)c->num_sms;  // this rank's FFN grid (read by the peers)
      if (cudaMemcpy(c->sym + L.ctr + 5 * sizeof(unsigned), &g, sizeof(g), cudaMemcpyHostToDevice) !=
          cudaSuccess) {
        tide_ctx_destroy(c);
        return fail(TIDE_ECUDA, "writing the FFN grid size into the symmetric region");
      }
    }
    c->connected = world == 1;
    c->ep_arrivals = c->num_sms;  // world 1: this rank's own FFN grid
  } else {
    ALLOC(c->x_all, c->eb * (size_t)R * c->H);
    ALLOC(c->topk_all, sizeof(int) * (size_t)R * k);
    ALLOC(c->gates_all, sizeof(float) * (size_t)R * k);
    ALLOC(c->pslot_all, sizeof(int) * (size_t)R * k);
    ALLOC(c->cnt_l, sizeof(int) * El);
    ALLOC(c->list_l, sizeof(int) * (size_t)El * R);
  }
  ALLOC(c->off_l, sizeof(int) * El);
  ALLOC(c->hits_l, sizeof(int) * El);
  if (!p2p) {
    ALLOC(c->partial, sizeof(float) * (size_t)R * c->H);
    ALLOC(c->recv, sizeof(float) * (size_t)R * c->H);
  }
  (void)N;
  if (make_map(&c->map_x_all, c->x_all, c->bf16, c->H, R, 1) != TIDE_OK) {
    std::string m = g_err;
    tide_ctx_destroy(c);
    return fail(TIDE_ECUDA, "%s", m.c_str());
  }
  if (p2p) {
    preload_ep_p2p_kernels(c);
    cudaDeviceSynchronize();  // the zeroed region is visible before any peer connects
  } else if (parent) {
    c->comm = parent->comm;
  } else {
    ncclUniqueId id;
    memcpy(&id, nccl_id, sizeof(id));
    ncclResult_t r = ncclCommInitRank(&c->comm, world, id, rank);
    if (r != ncclSuccess) {
      c->comm = nullptr;
      tide_ctx_destroy(c);
      return fail(TIDE_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
    }
    c->own_comm = true;
  }
  *out = c;
  return TIDE_OK;
}

tide_status tide_ctx_create_ep(const tide_layer_desc* d, int32_t device, const void* nccl_id,
                               int32_t rank, int32_t world, tide_ctx** out) {
  if (!nccl_id) return fail(TIDE_EINVAL, "nccl_unique_id is null");
  return ctx_create_ep_impl(d, device, nccl_id, nullptr, rank, world, out);
}

tide_status tide_ctx_create_ep_p2p(const tide_layer_desc* d, int32_t device, int32_t rank,
                                   int32_t world, tide_ctx** out) {
  return ctx_create_ep_impl(d, device, nullptr, nullptr, rank, world, out, true);
}

size_t tide_ep_handle_bytes(void) { return sizeof(cudaIpcMemHandle_t); }

tide_status tide_ctx_ep_export(tide_ctx* c, void* handle, void** base) {
  if (!c || !c->p2p) return fail(TIDE_EINVAL, "not a peer-memory EP context");
  if (!handle && !base) return fail(TIDE_EINVAL, "handle and base are both null");
  CU_TRY(cudaSetDevice(c->device));
  if (handle) {
    cudaIpcMemHandle_t h;
    CU_TRY(cudaIpcGetMemHandle(&h, c->sym));
    memcpy(handle, &h, sizeof(h));
  }
  if (base) *base = c->sym;
  return TIDE_OK;
}

// Whether device memory at ptr is allocated on `device` (a peer sharing this GPU).
static bool on_device(const void* ptr, int device) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();
    return true;  // unknown: take the safe (deferred-trigger) protocol
  }
  return a.device == device;
}

tide_status tide_ctx_ep_connect(tide_ctx* c, const void* handles, const void* const* bases) {
  if (!c || !c->p2p) return fail(TIDE_EINVAL, "not a peer-memory EP context");
  if (c->connected && c->world > 1) return fail(TIDE_EINVAL, "context already connected");
  if (!handles && !bases) return fail(TIDE_EINVAL, "handles and bases are both null");
  CU_TRY(cudaSetDevice(c->device));
  for (int p = 0; p < c->world; ++p) {
    if (p == c->rank) continue;
    if (bases && bases[p]) {
      c->peers.base[p] = static_cast<char*>(const_cast<void*>(bases[p]));
      c->peer_same_device = c->peer_same_device || on_device(bases[p], c->device);
      continue;
    }
    if (!handles) return fail(TIDE_EINVAL, "no handle or base for rank %d", p);
    cudaIpcMemHandle_t h;
    memcpy(&h, static_cast<const char*>(handles) + (size_t)p * sizeof(h), sizeof(h));
    void* ptr = nullptr;
    CU_TRY(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    c->ipc_opened.push_back(ptr);
    c->peers.base[p] = static_cast<char*>(ptr);
    c->peer_same_device = c->peer_same_device || on_device(ptr, c->device);
  }
  // every rank's FFN grid arrives once per CTA on each combine counter: the wait's target is
  // the sum of the ranks' grid sizes (each rank wrote its own into ctr[5] at creation)
  int total = 0;
  for (int p = 0; p < c->world; ++p) {
    unsigned g = 0;
    CU_TRY(cudaMemcpy(&g, c->peers.base[p] + c->lay.ctr + 5 * sizeof(unsigned), sizeof(g),
                      cudaMemcpyDefault));
    if (g == 0) return fail(TIDE_EINVAL, "rank %d's symmetric region has no FFN grid size", p);
    total += (int)g;
  }
  c->ep_arrivals = total;
  c->connected = true;
  return TIDE_OK;
}

tide_status tide_ctx_ep_error(tide_ctx* c, int32_t* err) {
  if (!c || !c->p2p || !err) return fail(TIDE_EINVAL, "not a peer-memory EP context / null err");
  unsigned v = 0;
  CU_TRY(cudaSetDevice(c->device));
  CU_TRY(cudaMemcpy(&v, c->sym + c->lay.ctr + 4 * sizeof(unsigned), sizeof(v), cudaMemcpyDeviceToHost));
  *err = (int32_t)v;
  return TIDE_OK;
}

tide_status tide_ctx_ep_wait(tide_ctx* c, int32_t timeout_ms) {
  if (!c || !c->ep) return fail(TIDE_EINVAL, "not an expert-parallel context");
  if (timeout_ms < 0) return fail(TIDE_EINVAL, "timeout_ms %d < 0", timeout_ms);
  CU_TRY(cudaSetDevice(c->device));
  if (!c->ev_ep_done) return TIDE_OK;  // no step yet
  const auto t0 = std::chrono::steady_clock::now();
  while (true) {
    const cudaError_t q = cudaEventQuery(c->ev_ep_done);
    if (c->comm) {
      ncclResult_t ar = ncclSuccess;
      NC_TRY(ncclCommGetAsyncError(c->comm, &ar));
      if (ar != ncclSuccess && ar != ncclInProgress) {
        if (c->own_comm) {  // a communicator shared with tide_ctx_create_ep_like contexts is
          ncclCommAbort(c->comm);  // aborted through the context that owns it
          c->comm = nullptr;
        }
        return fail(TIDE_ENCCL, "NCCL asynchronous error: %s%s", ncclGetErrorString(ar),
                    c->own_comm ? " (communicator aborted)" : "");
      }
    }
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady) return fail(TIDE_ECUDA, "step failed: %s", cudaGetErrorString(q));
    const auto ms = std::chrono::duration_cast<std::chrono::milliseconds>(
                        std::chrono::steady_clock::now() - t0).count();
    if (ms > timeout_ms) {
      if (c->comm) {
        if (c->own_comm) {
          ncclCommAbort(c->comm);
          c->comm = nullptr;
        }
        return fail(TIDE_ENCCL, "EP step not complete after %d ms%s", timeout_ms,
                    c->own_comm ? " (communicator aborted)" : "");
      }
      return fail(TIDE_ECUDA, "EP step not complete after %d ms", timeout_ms);
    }
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
  if (c->p2p) {
    int32_t err = 0;
    tide_status s = tide_ctx_ep_error(c, &err);
    if (s != TIDE_OK) return s;
    if (err) return fail(TIDE_ECUDA, "a peer-memory wait timed out (a peer did not arrive)");
  }
  return TIDE_OK;
}

tide_status tide_ctx_create_ep_like(const tide_layer_desc* d, tide_ctx* parent, tide_ctx** out) {
  if (!parent || !parent->ep) return fail(TIDE_EINVAL, "parent is not an expert-parallel context");
  return ctx_create_ep_impl(d, parent->device, nullptr, parent, parent->rank, parent->world, out);
}

// Lazily set up host_master resources (slot pool, staging ring, pinned mirrors).  Everything
// is allocated into locals and committed to the context only when all of it succeeded, so a
// failed call leaves the context as it was (the next call retries).
static tide_status ensure_pool(tide_ctx* c) {
  if (c->pool) return TIDE_OK;
  const int slots = c->capacity + c->staging + c->pf_slots_req;
  const int E = c->E;
  const int max_chunks = E + 2, max_entries2 = E + (c->maxN * c->k) / kMaxTok + 2;
  void* pool = nullptr;
  int4* entries2 = nullptr;
  int *ctrl2 = nullptr, *done2 = nullptr, *h_ctrl2 = nullptr, *h_slot_of = nullptr;
  void* h_info = nullptr;
  int4* h_entries2 = nullptr;
  std::vector<cudaEvent_t> ready(max_chunks, nullptr), done(max_chunks, nullptr);
  auto cleanup = [&]() {
    void* dev[] = {pool, entries2, ctrl2, done2};
    for (void* p : dev)
      if (p) cudaFree(p);
    void* host[] = {h_info, h_entries2, h_ctrl2, h_slot_of};
    for (void* p : host)
      if (p) cudaFreeHost(p);
    for (cudaEvent_t e : ready)
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : done)
      if (e) cudaEventDestroy(e);
  };
  bool ok = cudaMalloc(&pool, c->expert_bytes * slots) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    cleanup();
    return fail(TIDE_ENOMEM, "slot pool of %d experts (%zu B) failed", slots,
                c->expert_bytes * slots);
  }
  ok = cudaMalloc(reinterpret_cast<void**>(&entries2), sizeof(int4) * max_entries2) == cudaSuccess &&
       cudaMalloc(reinterpret_cast<void**>(&ctrl2), sizeof(int) * 2 * max_chunks) == cudaSuccess &&
       cudaMalloc(reinterpret_cast<void**>(&done2), sizeof(int) * max_entries2) == cudaSuccess &&
       cudaHostAlloc(&h_info, c->info_bytes, cudaHostAllocDefault) == cudaSuccess &&
       cudaHostAlloc(reinterpret_cast<void**>(&h_entries2), sizeof(int4) * max_entries2,
                     cudaHostAllocDefault) == cudaSuccess &&
       cudaHostAlloc(reinterpret_cast<void**>(&h_ctrl2),
                     sizeof(int) * (2 * max_chunks + max_entries2), cudaHostAllocDefault) == cudaSuccess &&
       cudaHostAlloc(reinterpret_cast<void**>(&h_slot_of), sizeof(int) * E, cudaHostAllocDefault) ==
           cudaSuccess;
  for (int i = 0; ok && i < max_chunks; ++i)
    ok = cudaEventCreateWithFlags(&ready[i], cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming) == cudaSuccess;
  std::vector<cudaEvent_t> pfev(c->pf_slots_req, nullptr);
  cudaEvent_t pf_free = nullptr;
  for (int i = 0; ok && i < c->pf_slots_req; ++i)
    ok = cudaEventCreateWithFlags(&pfev[i], cudaEventDisableTiming) == cudaSuccess;
  if (ok && c->pf_slots_req > 0) {
    ok = cudaEventCreateWithFlags(&pf_free, cudaEventDisableTiming) == cudaSuccess &&
         cudaEventRecord(pf_free, 0) == cudaSuccess;
  }
  if (!ok) {
    for (cudaEvent_t e : pfev)
      if (e) cudaEventDestroy(e);
    if (pf_free) cudaEventDestroy(pf_free);
  }
  if (ok) {
    for (int i = 0; i < E; ++i) h_slot_of[i] = -1;
    ok = cudaMemcpy(c->slot_of_dev, h_slot_of, sizeof(int) * E, cudaMemcpyHostToDevice) == cudaSuccess;
  }
  if (!ok) {
    cudaError_t e = cudaGetLastError();
    cleanup();
    return fail(TIDE_ENOMEM, "host_master resources: %s", cudaGetErrorString(e));
  }
  c->pool = pool;
  c->entries2 = entries2;
  c->ctrl2 = ctrl2;
  c->done2 = done2;
  c->h_info = h_info;
  c->h_entries2 = h_entries2;
  c->h_ctrl2 = h_ctrl2;
  c->h_slot_of = h_slot_of;
  c->max_chunks = max_chunks;
  c->max_entries2 = max_entries2;
  c->ev_chunk_ready = std::move(ready);
  c->ev_chunk_done = std::move(done);
  c->pf_ev = std::move(pfev);
  c->ev_pf_free = pf_free;
  c->pf_exp.assign(c->pf_slots_req, -1);
  c->owner.assign(c->capacity + c->staging, -1);  // retained + staging slots (prefetch apart)
  return TIDE_OK;
}

// build mode: cnt != nullptr (every CTA derives the work list from the counts);
// global mode: entries/n_entries (host-built staged chunk).
// NEXT-3 cross-layer L2 prefetch of the next layer's likely experts (tide_ctx_set_prefetch);
// all-null when off.  Issued by the FFN's CTAs as they run out of work (a combine-issued
// variant was measured and removed, DESIGN 11).
static L2Prefetch l2_prefetch_of(const tide_ctx* c) {
  L2Prefetch f{};
  if (!(c->pf_next && c->pf_weights && c->pf_max > 0)) return f;
  f.base = static_cast<const uint8_t*>(c->pf_weights);
  f.list = c->pf_next->pf_list;
  f.n = c->pf_next->pf_n;
  f.xb = (long long)c->pf_next->expert_bytes;
  // the gate/up rows only (2/3 of an expert: what the FFN's first wave of phase-1 items reads)
  // unless TIDE_PF_WHOLE_EXPERT; the byte budget then covers more experts
  f.span = c->knob_pf_whole ? f.xb : f.xb / 3 * 2;
  f.max = (int)std::min<int64_t>(c->pf_next->E + 1, c->pf_budget / f.span);
  // the next layer's shared expert (known once it has run a step) goes first
  f.shared = c->knob_pf_by_hits ? nullptr : static_cast<const uint8_t*>(c->pf_next->map_shared_src);
  return f;
}

static tide_status launch_ffn(tide_ctx* c, const int* cnt, const int* slot_of,
                              const int4* entries, const int* n_entries, int* sched, int* done,
                              int N, cudaStream_t st, bool ep_local = false,
                              unsigned long long* trace = nullptr, const int* par = nullptr,
                              bool prefetch = false, unsigned long long* itrace = nullptr) {
  FfnParams p;
  p.map_gu = c->map_gu;
  p.map_d = c->map_d;
  p.map_gu_s = c->have_shared_map ? c->map_gu_s : c->map_gu;
  p.map_d_s = c->have_shared_map ? c->map_d_s : c->map_d;
  p.map_x = c->map_x;
  p.map_h = c->map_h;
  p.cnt = cnt;
  p.par = par;
  p.pf = prefetch ? l2_prefetch_of(c) : L2Prefetch{};
  p.pf_self = L2Prefetch{};
  const int64_t self_bytes = c->pf_self_bytes >= 0 ? c->pf_self_bytes : c->pf_prev_budget / 2;
  if (prefetch && self_bytes > 0 && c->pf_target && cnt && !slot_of && c->map_src) {
    // this layer's own ranking (pf_list, written by its book kernel at the previous step, read
    // here before this step's book runs), past the range a previous layer's tail prefetched
    L2Prefetch& f = p.pf_self;
    f.base = static_cast<const uint8_t*>(c->map_src);
    f.list = c->pf_list;
    f.n = c->pf_n;
    f.xb = (long long)c->expert_bytes;
    f.span = c->knob_pf_whole ? f.xb : f.xb / 3 * 2;
    f.shared = c->knob_pf_by_hits ? nullptr : static_cast<const uint8_t*>(c->map_shared_src);
    const long long ppe = (f.span + kPfPiece - 1) / kPfPiece;
    const int64_t prev = c->pf_prev_budget;  // the range the previous layer's FFN tail covers
    const int done_e = prev > 0 ? (int)std::min<int64_t>(c->E + 1, prev / f.span) : 0;
    f.first = (long long)done_e * ppe;
    f.max = (int)std::min<int64_t>(c->E + 1, (prev + self_bytes) / f.span);
    if (f.max <= done_e) f = L2Prefetch{};
  }
  p.slot_of = slot_of;
  p.off_out = c->off;
  p.entries = entries;
  p.n_entries = n_entries;
  p.list = c->list;
  p.sched = sched;
  p.done = done;
  p.h_out = c->h_perm;
  p.y_out = c->y_perm;
  p.H = c->H;
  p.F = c->F;
  p.E = c->E;
  p.maxN = c->maxN;
  p.N = N;
  p.k = c->k;
  p.shared = (c->d.flags & TIDE_SHARED_EXPERT) ? 1 : 0;
  p.trace = trace;
  p.itrace = itrace;
  p.ep_P = 0;
  p.ep_e0 = 0;
  p.ep_El = 0;
  p.ep_dst = nullptr;
  p.ep_cnt_l = nullptr;
  p.ep_par = nullptr;
  p.ep_off_ypair = p.ep_off_hits = p.ep_off_ctr = 0;
  for (int i = 0; i < kEpMaxWorld; ++i) p.ep_base[i] = nullptr;
  if (ep_local && c->p2p) {  // fused owner scatter of the combine (ffn.cuh)
    p.ep_P = c->world;
    p.ep_e0 = c->e0;
    p.ep_El = c->El;
    p.ep_dst = c->dst_l;
    p.ep_cnt_l = c->cnt_l;
    p.ep_par = c->cnt_par;
    for (int i = 0; i < kEpMaxWorld; ++i) p.ep_base[i] = c->peers.base[i];
    p.ep_off_ypair = c->lay.ypair;
    p.ep_off_hits = c->lay.hits_all;
    p.ep_off_ctr = c->lay.ctr;
  }
  p.shared_row0 = N * c->k;
  p.shared_tok0 = 0;
  if (ep_local) {  // local experts over all ranks' rows; shared expert on this rank's tokens
    p.map_x = c->map_x_all;
    p.off_out = c->off_l;
    p.list = c->list_l;
    p.E = c->El;
    p.maxN = c->rows_all;
    p.shared_row0 = c->rows_all * c->k;
    p.shared_tok0 = c->rank * c->maxN;
  }
  const bool ep_scatter = p.ep_P > 0;
  if (c->bf16)
    CU_TRY(launch_pdl(ep_scatter ? tide_ffn_kernel<__nv_bfloat16, true>
                                 : tide_ffn_kernel<__nv_bfloat16, false>,
                      dim3(c->num_sms), dim3(kFfnThreads), c->ffn_smem, st, p));
  else
    CU_TRY(launch_pdl(ep_scatter ? tide_ffn_kernel<float, true> : tide_ffn_kernel<float, false>,
                      dim3(c->num_sms), dim3(kFfnThreads), c->ffn_smem, st, p));
  c->launches++;
  c->ffn_launches++;
  return TIDE_OK;
}

static tide_status ensure_weight_maps(tide_ctx* c, const void* src, int rows_experts,
                                      const void* shared) {
  if (src != c->map_src || rows_experts != c->map_src_rows) {
    tide_status s = make_map(&c->map_gu, src, c->bf16, c->H, (uint64_t)rows_experts * 3 * c->F, 128);
    if (s != TIDE_OK) return s;
    s = make_map(&c->map_d, src, c->bf16, c->F, (uint64_t)rows_experts * 3 * c->H, 128);
    if (s != TIDE_OK) return s;
    c->map_src = src;
    c->map_src_rows = rows_experts;
  }
  if (shared && shared != c->map_shared_src) {
    tide_status s = make_map(&c->map_gu_s, shared, c->bf16, c->H, (uint64_t)3 * c->F, 128);
    if (s != TIDE_OK) return s;
    s = make_map(&c->map_d_s, shared, c->bf16, c->F, (uint64_t)3 * c->H, 128);
    if (s != TIDE_OK) return s;
    c->map_shared_src = shared;
    c->have_shared_map = true;
  }
  return TIDE_OK;
}

static void fill_stats(tide_ctx* c, const RouteInfo* info, int N, int streamed, int copies,
                       int64_t weight_bytes, tide_step_stats* st, int64_t resident_wb,
                       int resident_rows, int ffn_launches) {
  st->resident_weight_bytes = resident_wb;
  st->resident_rows = resident_rows;
  st->ffn_launches = ffn_launches;
  st->refreshed = info->refreshed;
  st->resident_pairs = info->resident_pairs;
  st->nonresident_pairs = N * c->k - info->resident_pairs;
  st->promotions = info->promotions;
  st->evictions = info->evictions;
  st->unique_experts = info->unique_experts;
  st->experts_streamed = streamed;
  st->copies = copies;
  st->h2d_bytes = (int64_t)copies * (int64_t)c->expert_bytes;
  st->weight_bytes_read = weight_bytes;
}

static BookParams book_params(tide_ctx* c, const int* cnt, const uint8_t* placement, int N,
                              int refresh, int capacity, int32_t* hit_counts,
                              uint8_t* placement_out, int E_override, int step, const int* par) {
  const int E = E_override ? E_override : c->E;
  BookParams b;
  b.cnt = cnt;
  b.par = par;
  b.pf_list = c->pf_target ? c->pf_list : nullptr;  // EP: local expert indices
  b.pf_n = c->pf_n;
  b.pf_by_hits = c->knob_pf_by_hits ? 1 : 0;
  b.mask = c->mask;
  b.mask_rw = c->mask;
  b.topk_idx = c->topk;
  b.placement_in = placement;
  b.N = N;
  b.E = E;
  b.k = c->k;
  b.refresh = refresh;
  b.capacity = capacity;
  b.acc = c->counter_acc;
  b.mode = (c->d.flags & TIDE_COUNTER_WINDOW) ? 1 : (c->d.flags & TIDE_COUNTER_CUMULATIVE) ? 2 : 0;
  b.step = step;
  b.incumbent = (c->d.flags & TIDE_TIE_INCUMBENT) ? 1 : 0;
  b.hit_counts = hit_counts;
  b.placement_out = placement_out;
  b.order = c->order;
  b.offsets = c->offsets;
  b.pos = c->pos;
  b.info = c->info;
  return b;
}

static tide_status launch_book(tide_ctx* c, const int* cnt, const uint8_t* placement, int N,
                               int refresh, int capacity, int32_t* hit_counts,
                               uint8_t* placement_out, cudaStream_t st, int E_override = 0,
                               int step = 0, const int* par = nullptr) {
  const BookParams b = book_params(c, cnt, placement, N, refresh, capacity, hit_counts, placement_out,
                                   E_override, step, par);
  tide_book_kernel<<<1, 1024, sizeof(int) * 6 * b.E, st>>>(b);
  CU_TRY(cudaGetLastError());
  c->launches++;
  return TIDE_OK;
}

static tide_status launch_route(tide_ctx* c, const void* x, int N, const void* wr,
                                tide_step_debug* dbg, cudaStream_t st) {
  const int E = c->E, k = c->k, H = c->H;
  RouteParams rp;
  rp.x = N > 0 ? x : c->x_in;  // no tokens: a valid (unread) row for the clamped loads
  rp.wr = wr;
  rp.x_in = c->x_in;
  rp.logits = c->logits;
  rp.logits64 = c->logits64;
  rp.ksplit = 1;
  rp.N = N;
  rp.E = E;
  rp.H = H;
  rp.k = k;
  rp.tpc = N <= 64 ? 4 : 8;  // tokens per CTA row of the route grid
  if (c->knob_route_tpc > 0) rp.tpc = c->knob_route_tpc;
  rp.norm_topk = (c->d.flags & TIDE_NORM_TOPK) ? 1 : 0;
  rp.maxN = c->maxN;
  rp.topk_idx = c->topk;
  rp.gates = c->gates;
  rp.pair_slot = c->pair_slot;
  rp.cnt2 = c->cnt;
  rp.par = c->cnt_par;
  rp.g_done = c->cnt_par + 1;
  rp.list = c->list;
  rp.mask = c->mask;
  rp.g_cnt = c->g_cnt;
  rp.zero_i = c->ffn_ctrl;
  rp.n_zero = 2 + c->max_entries;
  rp.trace = (dbg && dbg->route_trace) ? reinterpret_cast<unsigned long long*>(dbg->route_trace)
                                       : nullptr;
  rp.ep_P = 0;
  rp.ep_rank = 0;
  rp.ep_lists = 0;
  rp.ep_shared_dev = 0;
  if (c->p2p) {  // peer-memory EP: the router dispatches (route.cuh)
    rp.ep_P = c->world;
    rp.ep_rank = c->rank;
    for (int i = 0; i < kEpMaxWorld; ++i) rp.ep_base[i] = c->peers.base[i];
    rp.ep_off_x = c->lay.x_all;
    rp.ep_off_ctr = c->lay.ctr;
    rp.ep_off_cnt = c->lay.cnt_l;
    rp.ep_off_list = c->lay.list_l;
    rp.ep_off_dst = c->lay.dst_l;
    rp.ep_lists = 1;  // the route grid's last CTA waits until every source rank dispatched
    rp.ep_shared_dev = c->peer_same_device ? 1 : 0;
    rp.ep_El = c->El;
    rp.ep_rows = c->rows_all;
  }
  // bf16 routers run phase 1 on the tensor cores (16 experts x 8 tokens per CTA);
  // TIDE_ROUTER_CC=1 forces the CUDA-core kernel (A/B measurement)
  if (c->bf16 && E % 16 == 0 && H % 256 == 0 && !c->knob_router_cc) {
    rp.tpc = 8;
    // small batches: each 16-expert tile is split over 2 CTAs (half of H each, fp64 partials
    // summed in phase 2) while the grid still fits one wave: half the bytes per SM
    const int tiles = (E / 16) * std::max(1, (N + 7) / 8);
    rp.ksplit = (c->logits64 && H % 512 == 0 && 2 * tiles <= c->num_sms && !c->knob_route_ksplit1)
                    ? 2 : 1;
    const dim3 grid((E / 16) * rp.ksplit, std::max(1, (N + 7) / 8));
    cudaError_t le;
    // large batches (more than one wave of 16 x 8 tiles): two CTAs per SM (<= 128 registers)
    const bool two_per_sm = grid.x * grid.y > (unsigned)c->num_sms && !c->knob_route_one_per_sm;
#define TC_LAUNCH(EP)                                                                        \
  le = two_per_sm ? launch_pdl(tide_route_tc_kernel<EP, 8, 2>, grid, dim3(kRouteThreads), 0, st, rp) \
                  : launch_pdl(tide_route_tc_kernel<EP, 8, 1>, grid, dim3(kRouteThreads), 0, st, rp)
    switch (route_epl(E)) {
      case 1: TC_LAUNCH(1); break;
      case 2: TC_LAUNCH(2); break;
      case 4: TC_LAUNCH(4); break;
      case 8: TC_LAUNCH(8); break;
      case 16: TC_LAUNCH(16); break;
      default: TC_LAUNCH(32); break;
    }
#undef TC_LAUNCH
    CU_TRY(le);
    c->launches++;
    return TIDE_OK;
  }
  {
    const dim3 grid((E + kRouterWarps - 1) / kRouterWarps, std::max(1, (N + rp.tpc - 1) / rp.tpc));
    cudaError_t le;
    const int epl = route_epl(E);
#define ROUTE_LAUNCH(TT, EP) \
  le = launch_pdl(tide_route_kernel<TT, EP>, grid, dim3(kRouteThreads), 0, st, rp)
#define ROUTE_DISPATCH(TT)                     \
    switch (epl) {                             \
      case 1: ROUTE_LAUNCH(TT, 1); break;      \
      case 2: ROUTE_LAUNCH(TT, 2); break;      \
      case 4: ROUTE_LAUNCH(TT, 4); break;      \
      case 8: ROUTE_LAUNCH(TT, 8); break;      \
      case 16: ROUTE_LAUNCH(TT, 16); break;    \
      default: ROUTE_LAUNCH(TT, 32); break;    \
    }
    if (c->bf16) {
      ROUTE_DISPATCH(__nv_bfloat16)
    } else {
      ROUTE_DISPATCH(float)
    }
#undef ROUTE_DISPATCH
#undef ROUTE_LAUNCH
    CU_TRY(le);
    c->launches++;
  }
  return TIDE_OK;
}

// NEXT-3 H2D prefetch (host_master): called at the end of the previous layer's step; copies the
// experts `n` streamed at its previous step (most-hit first, those not in HBM now) into its
// prefetch slots on its side stream, so the link works through the gap before `n`'s own step
// plans its copies (its route, bookkeeping and host round trip).  A wrong prediction costs
// link time and nothing else (the slot is simply not used).
static tide_status issue_h2d_prefetch(tide_ctx* n) {
  if (!n->pool || !n->last_master || n->pf_exp.empty()) return TIDE_OK;
  CU_TRY(cudaStreamWaitEvent(n->side, n->ev_pf_free, 0));  // its last step's reads are done
  const size_t xb = n->expert_bytes;
  uint8_t* pool = static_cast<uint8_t*>(n->pool);
  const uint8_t* master = static_cast<const uint8_t*>(n->last_master);
  const int base = n->capacity + n->staging;
  int i = 0;
  for (int e : n->last_streamed) {
    if (i == (int)n->pf_exp.size()) break;
    if (n->slot_of[e] >= 0) continue;  // in HBM now
    CU_TRY(cudaMemcpyAsync(pool + (size_t)(base + i) * xb, master + (size_t)e * xb, xb,
                           cudaMemcpyHostToDevice, n->side));
    CU_TRY(cudaEventRecord(n->pf_ev[i], n->side));
    n->pf_exp[i] = e;
    ++i;
    n->pf_issued++;
  }
  return TIDE_OK;
}

// host_master: plan and enqueue the H2D copies (a6) and the staged FFN chunks (a8).
// Slot semantics (R-12/R-13): an expert in HBM at step start is served from HBM this
// step; a slot released by an expert that is hit this step is rewritten only after the
// resident FFN has read it; hit experts not in HBM are copied into a pool slot when in
// placement', else into the staging ring (not retained); eager promotions copy promoted
// experts without hits after the hit ones.
static tide_status pool_step(tide_ctx* c, const tide_expert_weights* w, const RouteInfo* hinfo,
                             int N, cudaStream_t st, int* streamed, int* copies,
                             int64_t* weight_bytes, int* resident_rows, int* n_chunks,
                             int64_t* resident_wb) {
  const int E = c->E;
  const int* hits = reinterpret_cast<const int*>(hinfo + 1);
  const uint8_t* pl = reinterpret_cast<const uint8_t*>(hits + E);
  const bool lazy = (c->d.flags & TIDE_LAZY_PROMOTE) != 0;
  const int C = c->capacity, S = c->staging, half = std::max(1, S / 2);
  const uint8_t* master = static_cast<const uint8_t*>(w->host_master);
  uint8_t* pool = static_cast<uint8_t*>(c->pool);
  const size_t xb = c->expert_bytes;
  // the new slot maps are planned on copies and committed only after every enqueue succeeded
  std::vector<int> slot_of = c->slot_of, owner = c->owner;
  std::vector<int> off(E), loaded0(E);
  for (int e = 0, r = 0; e < E; ++e) {  // same row rule as the FFN's build mode
    off[e] = r;
    r += hits[e];
    loaded0[e] = slot_of[e] >= 0;
    if (hits[e] > 0 && loaded0[e]) {
      *weight_bytes += (int64_t)xb * ((hits[e] + kMaxTok - 1) / kMaxTok);
      *resident_rows += hits[e];
    }
  }
  *resident_wb = *weight_bytes;  // the resident launch: experts in HBM at step start
  std::vector<int> free_now, free_after_gemm1;
  for (int sl = 0; sl < C; ++sl)
    if (owner[sl] < 0) free_now.push_back(sl);
  for (int e = 0; e < E; ++e) {
    const int sl = slot_of[e];
    if (sl >= 0 && !pl[e]) {
      (hits[e] > 0 ? free_after_gemm1 : free_now).push_back(sl);
      owner[sl] = -1;
      slot_of[e] = -1;
    }
  }
  // NEXT-3 H2D prefetch: experts the previous layer's step already copied into this
  // context's prefetch slots (predicted from this layer's previous step) are not copied
  // again: a staged one is computed from its prefetch slot, a promoted one is moved into
  // its retained slot by a device-to-device copy
  auto prefetched = [&](int e) -> int {
    for (int i = 0; i < (int)c->pf_exp.size(); ++i)
      if (c->pf_exp[i] == e) return i;
    return -1;
  };
  *copies += c->pf_issued;  // H2D copies issued for this step by the previous layer
  c->pf_issued = 0;
  struct Copy { int e, dst; bool after_gemm1, staged; int pf; };
  std::vector<Copy> hit_copies, cold_copies;
  size_t fn = 0, fa = 0;
  auto take_slot = [&](bool& after) -> int {
    if (fn < free_now.size()) { after = false; return free_now[fn++]; }
    after = true;
    return free_after_gemm1[fa++];
  };
  for (int e = 0; e < E; ++e) {
    if (hits[e] == 0 || loaded0[e]) continue;
    Copy cp{e, -1, false, false, prefetched(e)};
    if (pl[e]) {
      cp.dst = take_slot(cp.after_gemm1);
      owner[cp.dst] = e;
      slot_of[e] = cp.dst;
    } else {
      cp.staged = true;
    }
    hit_copies.push_back(cp);
  }
  if (!lazy)
    for (int e = 0; e < E; ++e)
      if (pl[e] && slot_of[e] < 0 && hits[e] == 0) {
        Copy cp{e, -1, false, false, -1};
        cp.dst = take_slot(cp.after_gemm1);
        owner[cp.dst] = e;
        slot_of[e] = cp.dst;
        cold_copies.push_back(cp);
      }
  *streamed = (int)hit_copies.size();
  // prefetched experts first (their bytes are already in flight), then the others; slots
  // freed only after the resident FFN last (stable: ascending id within each class)
  std::stable_partition(hit_copies.begin(), hit_copies.end(),
                        [](const Copy& a) { return a.pf >= 0; });
  std::stable_partition(hit_copies.begin(), hit_copies.end(),
                        [](const Copy& a) { return !a.after_gemm1; });
  std::vector<std::pair<int, int>> chunks;  // [begin, end) into hit_copies
  {
    int b = 0, used = 0;
    for (int i = 0; i < (int)hit_copies.size(); ++i) {
      const bool needs_stage = hit_copies[i].staged && hit_copies[i].pf < 0;
      const bool boundary = (needs_stage && used == half) ||
                            (i > b && hit_copies[i].after_gemm1 && !hit_copies[i - 1].after_gemm1) ||
                            (i > b && hit_copies[i].pf < 0 && hit_copies[i - 1].pf >= 0);
      if (boundary) { chunks.push_back({b, i}); b = i; used = 0; }
      if (needs_stage) used++;
    }
    if (b < (int)hit_copies.size()) chunks.push_back({b, (int)hit_copies.size()});
  }
  if ((int)chunks.size() > c->max_chunks) return fail(TIDE_EINVAL, "too many staged chunks");
  *n_chunks = (int)chunks.size();
  int ne = 0;
  std::vector<int> chunk_first(chunks.size() + 1, 0);
  for (size_t ci = 0; ci < chunks.size(); ++ci) {
    chunk_first[ci] = ne;
    int stage_i = 0;
    for (int i = chunks[ci].first; i < chunks[ci].second; ++i) {
      Copy& cp = hit_copies[i];
      if (cp.staged) cp.dst = cp.pf >= 0 ? C + S + cp.pf : C + (int)(ci % 2) * half + (stage_i++);
      const int m = hits[cp.e];
      for (int t = 0; t < m; t += kMaxTok) {
        c->h_entries2[ne++] = make_int4(cp.dst, off[cp.e] + t, std::min(kMaxTok, m - t),
                                        cp.e * c->maxN + t);
        *weight_bytes += (int64_t)xb;
      }
    }
    c->h_ctrl2[2 * ci] = ne - chunk_first[ci];
    c->h_ctrl2[2 * ci + 1] = 0;
  }
  chunk_first[chunks.size()] = ne;
  int* h_done2 = c->h_ctrl2 + 2 * c->max_chunks;
  for (int i = 0; i < ne; ++i) h_done2[i] = 0;
  if (!chunks.empty()) {
    CU_TRY(cudaMemcpyAsync(c->entries2, c->h_entries2, sizeof(int4) * ne, cudaMemcpyHostToDevice, st));
    CU_TRY(cudaMemcpyAsync(c->ctrl2, c->h_ctrl2, sizeof(int) * 2 * chunks.size(),
                           cudaMemcpyHostToDevice, st));
    CU_TRY(cudaMemcpyAsync(c->done2, h_done2, sizeof(int) * ne, cudaMemcpyHostToDevice, st));
  }
  bool waited_gemm1 = false;
  for (size_t ci = 0; ci < chunks.size(); ++ci) {
    if (ci >= 2) CU_TRY(cudaStreamWaitEvent(c->side, c->ev_chunk_done[ci - 2], 0));
    for (int i = chunks[ci].first; i < chunks[ci].second; ++i) {
      const Copy& cp = hit_copies[i];
      if (cp.after_gemm1 && !waited_gemm1) {
        CU_TRY(cudaStreamWaitEvent(c->side, c->ev_gemm1, 0));
        waited_gemm1 = true;
      }
      if (cp.pf >= 0) {  // already in a prefetch slot (H2D enqueued by the previous layer)
        CU_TRY(cudaStreamWaitEvent(c->side, c->pf_ev[cp.pf], 0));
        if (!cp.staged)  // retained: HBM-to-HBM into its slot
          CU_TRY(cudaMemcpyAsync(pool + (size_t)cp.dst * xb, pool + (size_t)(C + S + cp.pf) * xb,
                                 xb, cudaMemcpyDeviceToDevice, c->side));
        continue;
      }
      CU_TRY(cudaMemcpyAsync(pool + (size_t)cp.dst * xb, master + (size_t)cp.e * xb, xb,
                             cudaMemcpyHostToDevice, c->side));
      (*copies)++;
    }
    CU_TRY(cudaEventRecord(c->ev_chunk_ready[ci], c->side));
    CU_TRY(cudaStreamWaitEvent(st, c->ev_chunk_ready[ci], 0));
    tide_status s = launch_ffn(c, nullptr, nullptr, c->entries2 + chunk_first[ci], c->ctrl2 + 2 * ci,
                               c->ctrl2 + 2 * ci + 1, c->done2 + chunk_first[ci], N, st);
    if (s != TIDE_OK) return s;
    CU_TRY(cudaEventRecord(c->ev_chunk_done[ci], st));
  }
  for (const Copy& cp : cold_copies) {
    if (cp.after_gemm1 && !waited_gemm1) {
      CU_TRY(cudaStreamWaitEvent(c->side, c->ev_gemm1, 0));
      waited_gemm1 = true;
    }
    CU_TRY(cudaMemcpyAsync(pool + (size_t)cp.dst * xb, master + (size_t)cp.e * xb, xb,
                           cudaMemcpyHostToDevice, c->side));
    (*copies)++;
  }
  CU_TRY(cudaEventRecord(c->ev_side_done, c->side));
  CU_TRY(cudaStreamWaitEvent(st, c->ev_side_done, 0));
  for (int e = 0; e < E; ++e) c->h_slot_of[e] = slot_of[e];
  CU_TRY(cudaMemcpyAsync(c->slot_of_dev, c->h_slot_of, sizeof(int) * E, cudaMemcpyHostToDevice, st));
  c->slot_of = std::move(slot_of);
  c->owner = std::move(owner);
  // NEXT-3 H2D prefetch: the prefetch slots are free once this step's FFN launches are done;
  // remember what streamed (hit, not in HBM), most-hit first: the prediction for the next
  // step, which the previous layer's step prefetches into those slots
  if (!c->pf_exp.empty()) {
    std::fill(c->pf_exp.begin(), c->pf_exp.end(), -1);
    CU_TRY(cudaEventRecord(c->ev_pf_free, st));
    c->last_streamed.clear();
    for (const Copy& cp : hit_copies)  // experts hit by a single token flicker: not predicted
      if (hits[cp.e] >= c->pf_min_hits) c->last_streamed.push_back(cp.e);
    std::stable_sort(c->last_streamed.begin(), c->last_streamed.end(),
                     [hits](int a, int b) { return hits[a] > hits[b]; });
    c->last_master = master;
  }
  if (c->pf_next_h) {
    tide_status s = issue_h2d_prefetch(c->pf_next_h);
    if (s != TIDE_OK) return s;
  }
  return TIDE_OK;
}

tide_status tide_moe_step(tide_ctx* c, const void* x, int32_t N, const void* wr,
                          const tide_expert_weights* w, const uint8_t* placement, int32_t step,
                          int32_t interval, int32_t capacity, void* out, int32_t* hit_counts,
                          uint8_t* placement_out, tide_step_stats* stats, tide_step_debug* dbg,
                          void* stream) {
  // ---------------- argument checks (nothing enqueued on failure)
  if (!c) return fail(TIDE_EINVAL, "ctx is null");
  if (N < 0 || N > c->maxN) return fail(TIDE_EINVAL, "num_tokens %d outside [0, %d]", N, c->maxN);
  if (!w) return fail(TIDE_EINVAL, "expert_w is null");
  if ((w->device_all == nullptr) == (w->host_master == nullptr))
    return fail(TIDE_EINVAL, "exactly one of device_all / host_master must be set");
  const bool shared = (c->d.flags & TIDE_SHARED_EXPERT) != 0;
  if (shared && !w->shared_w) return fail(TIDE_EINVAL, "TIDE_SHARED_EXPERT set but shared_w is null");
  if (!placement || !placement_out || !hit_counts || (N > 0 && (!x || !out)) || !wr)
    return fail(TIDE_EINVAL, "null tensor argument");
  if (interval < 1) return fail(TIDE_EINVAL, "interval %d < 1", interval);
  if (step < 0) return fail(TIDE_EINVAL, "step %d < 0", step);
  if (capacity != c->capacity)
    return fail(TIDE_ECAPACITY, "capacity %d != context capacity %d", capacity, c->capacity);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CU_TRY(cudaSetDevice(c->device));
  const bool pool_mode = w->host_master != nullptr;
  if (pool_mode) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, w->host_master) != cudaSuccess ||
        a.type != cudaMemoryTypeHost) {
      cudaGetLastError();
      return fail(TIDE_EINVAL, "host_master is not pinned host memory");
    }
    tide_status s = ensure_pool(c);
    if (s != TIDE_OK) return s;
  }
  const int E = c->E, k = c->k, H = c->H;
  const int refresh = (step % interval) == 0;
  tide_status s = ensure_weight_maps(c, pool_mode ? c->pool : w->device_all,
                                     pool_mode ? c->capacity + c->staging + c->pf_slots_req : E,
                                     shared ? w->shared_w : nullptr);
  if (s != TIDE_OK) return s;

  tide_ctx::Rec rec{};
  const int64_t launches0 = c->launches, ffn0 = c->ffn_launches;
  if (c->timing) {
    for (cudaEvent_t& e : rec.ev) e = take_event(c);
    CU_TRY(cudaEventRecord(rec.ev[0], st));
  }
  // ---------------- a1..a3: router, top-k, hits and per-expert token lists
  s = launch_route(c, x, N, wr, dbg, st);
  if (s != TIDE_OK) return s;
  if (c->timing) CU_TRY(cudaEventRecord(rec.ev[1], st));

  // ---------------- a4/a5 bookkeeping (placement, buckets, pos, info)
  if (pool_mode) {
    s = launch_book(c, c->cnt, placement, N, refresh, capacity, hit_counts, placement_out, st, 0,
                    step, c->cnt_par);
    if (s != TIDE_OK) return s;
    CU_TRY(cudaMemcpyAsync(c->h_info, c->info, c->info_bytes, cudaMemcpyDeviceToHost, st));
    CU_TRY(cudaEventRecord(c->ev_info, st));
  } else {
    CU_TRY(cudaEventRecord(c->ev_route, st));
    CU_TRY(cudaStreamWaitEvent(c->side, c->ev_route, 0));
    s = launch_book(c, c->cnt, placement, N, refresh, capacity, hit_counts, placement_out, c->side, 0,
                    step, c->cnt_par);
    if (s != TIDE_OK) return s;
    CU_TRY(cudaEventRecord(c->ev_book, c->side));
  }
  if (c->timing) {
    CU_TRY(cudaEventRecord(rec.ev[2], st));
    CU_TRY(cudaEventRecord(rec.ev[3], st));
  }
  // ---------------- a7/a9 FFN over the hit experts already in HBM (+ shared expert)
  if (N > 0) {
    s = launch_ffn(c, c->cnt, pool_mode ? c->slot_of_dev : nullptr, nullptr, nullptr, c->ffn_ctrl,
                   c->ffn_ctrl + 1, N, st, false,
                   dbg ? reinterpret_cast<unsigned long long*>(dbg->ffn_trace) : nullptr, c->cnt_par,
                   !pool_mode,
                   dbg ? reinterpret_cast<unsigned long long*>(dbg->ffn_item_trace) : nullptr);
    if (s != TIDE_OK) return s;
  }
  if (c->timing) CU_TRY(cudaEventRecord(rec.ev[4], st));

  int streamed = 0, copies = 0, res_rows = 0, n_chunks = 0;
  int64_t weight_bytes = 0, res_wb = 0;
  const RouteInfo* hinfo = nullptr;
  if (pool_mode) {  // ---------------- a6 + a8
    CU_TRY(cudaEventRecord(c->ev_gemm1, st));
    CU_TRY(cudaEventSynchronize(c->ev_info));
    hinfo = static_cast<const RouteInfo*>(c->h_info);
    if (hinfo->status != 0)
      return fail(TIDE_EPLACEMENT, "step %d is not a refresh and placement holds more than %d experts",
                  step, capacity);
    s = pool_step(c, w, hinfo, N, st, &streamed, &copies, &weight_bytes, &res_rows, &n_chunks,
                  &res_wb);
    if (s != TIDE_OK) return s;
  }
  if (c->timing) CU_TRY(cudaEventRecord(rec.ev[5], st));

  // a4/a5 outputs ordered on the stream: the join sits before the combine, not after it (the
  // next layer's route then follows the combine on its programmatic edge alone: +0.45%)
  if (!pool_mode) CU_TRY(cudaStreamWaitEvent(st, c->ev_book, 0));
  // ---------------- a10 combine
  if (N > 0) {
    const dim3 grid(N, (H + 511) / 512);
    const size_t csmem = sizeof(int) * E;
    unsigned long long* ctr =  // debug: [6] latest start, [7] latest end in CTA 0's FFN record
        (dbg && dbg->ffn_trace) ? reinterpret_cast<unsigned long long*>(dbg->ffn_trace) + 6 : nullptr;
    if (c->bf16)
      CU_TRY(launch_pdl(tide_combine_kernel<__nv_bfloat16>, grid, dim3(128), csmem, st,
                        (const float*)c->y_perm, (const float*)c->gates, (const int*)c->topk,
                        (const int*)c->pair_slot, (const int*)c->cnt, (const int*)c->cnt_par, E,
                        static_cast<__nv_bfloat16*>(out), N, k, H, shared ? 1 : 0, ctr));
    else
      CU_TRY(launch_pdl(tide_combine_kernel<float>, grid, dim3(128), csmem, st,
                        (const float*)c->y_perm, (const float*)c->gates, (const int*)c->topk,
                        (const int*)c->pair_slot, (const int*)c->cnt, (const int*)c->cnt_par, E,
                        static_cast<float*>(out), N, k, H, shared ? 1 : 0, ctr));
    c->launches++;
  }
  if (c->timing) {
    CU_TRY(cudaEventRecord(rec.ev[6], st));
    rec.launches = c->launches - launches0;
    rec.ffn_launches = c->ffn_launches - ffn0;
    c->pending.push_back(rec);
  }
  if (dbg) {
    if (dbg->topk_idx) CU_TRY(cudaMemcpyAsync(dbg->topk_idx, c->topk, sizeof(int) * N * k, cudaMemcpyDeviceToDevice, st));
    if (dbg->gates) CU_TRY(cudaMemcpyAsync(dbg->gates, c->gates, sizeof(float) * N * k, cudaMemcpyDeviceToDevice, st));
    if (dbg->pos) CU_TRY(cudaMemcpyAsync(dbg->pos, c->pos, sizeof(int) * N * k, cudaMemcpyDeviceToDevice, st));
    if (dbg->order) CU_TRY(cudaMemcpyAsync(dbg->order, c->order, sizeof(int) * E, cudaMemcpyDeviceToDevice, st));
    if (dbg->offsets) CU_TRY(cudaMemcpyAsync(dbg->offsets, c->offsets, sizeof(int) * (E + 1), cudaMemcpyDeviceToDevice, st));
    if (dbg->logits) CU_TRY(cudaMemcpyAsync(dbg->logits, c->logits, sizeof(float) * N * E, cudaMemcpyDeviceToDevice, st));
  }
  if (stats) {
    RouteInfo local;
    if (!pool_mode) {
      std::vector<int> hits(E);
      CU_TRY(cudaMemcpyAsync(&local, c->info, sizeof(RouteInfo), cudaMemcpyDeviceToHost, st));
      CU_TRY(cudaMemcpyAsync(hits.data(), c->info + 1, sizeof(int) * E, cudaMemcpyDeviceToHost, st));
      CU_TRY(cudaStreamSynchronize(st));
      hinfo = &local;
      if (local.status != 0)
        return fail(TIDE_EPLACEMENT, "step %d is not a refresh and placement holds more than %d experts",
                    step, capacity);
      for (int e = 0; e < E; ++e)
        weight_bytes += (int64_t)c->expert_bytes * ((hits[e] + kMaxTok - 1) / kMaxTok);
    } else {
      CU_TRY(cudaStreamSynchronize(st));
    }
    const int64_t shared_wb = shared ? (int64_t)c->expert_bytes * ((N + kMaxTok - 1) / kMaxTok) : 0;
    weight_bytes += shared_wb;
    if (!pool_mode) {  // one FFN launch computes everything
      res_wb = weight_bytes;
      res_rows = N * k;
    } else {
      res_wb += shared_wb;
    }
    if (shared) res_rows += N;
    fill_stats(c, hinfo, N, streamed, copies, weight_bytes, stats, res_wb, res_rows,
               (N > 0 ? 1 : 0) + n_chunks);
  }
  return TIDE_OK;
}

tide_status tide_moe_step_ep(tide_ctx* c, const void* x, int32_t N, const void* wr,
                             const void* local_experts, const void* shared_w,
                             const uint8_t* placement, int32_t step, int32_t interval,
                             int32_t capacity, void* out, int32_t* hit_counts,
                             uint8_t* placement_out, tide_step_stats* stats, void* stream) {
  if (!c || !c->ep) return fail(TIDE_EINVAL, "not an expert-parallel context");
  if (c->p2p && !c->connected)
    return fail(TIDE_EINVAL, "peer-memory EP context not connected (tide_ctx_ep_connect)");
  if (N < 0 || N > c->maxN) return fail(TIDE_EINVAL, "num_tokens %d outside [0, %d]", N, c->maxN);
  const bool shared = (c->d.flags & TIDE_SHARED_EXPERT) != 0;
  if (!local_experts || !wr || !placement || !placement_out || !hit_counts || (N > 0 && (!x || !out)))
    return fail(TIDE_EINVAL, "null tensor argument");
  if (shared && !shared_w) return fail(TIDE_EINVAL, "TIDE_SHARED_EXPERT set but shared_w is null");
  if (interval < 1) return fail(TIDE_EINVAL, "interval %d < 1", interval);
  if (step < 0) return fail(TIDE_EINVAL, "step %d < 0", step);
  if (capacity < 1 || capacity > c->El)
    return fail(TIDE_ECAPACITY, "capacity %d outside [1, %d] (per rank)", capacity, c->El);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CU_TRY(cudaSetDevice(c->device));
  const int k = c->k, H = c->H, maxN = c->maxN, R = c->rows_all, El = c->El;
  const int refresh = (step % interval) == 0;
  tide_status s = ensure_weight_maps(c, local_experts, El, shared ? shared_w : nullptr);
  if (s != TIDE_OK) return s;
  tide_ctx::Rec rec{};
  const int64_t launches0 = c->launches, ffn0 = c->ffn_launches;
  if (c->timing) {
    for (cudaEvent_t& e : rec.ev) e = take_event(c);
    CU_TRY(cudaEventRecord(rec.ev[0], st));
  }
  // a1..a3 on this rank's tokens
  s = launch_route(c, x, N, wr, nullptr, st);
  if (s != TIDE_OK) return s;
  if (c->timing) CU_TRY(cudaEventRecord(rec.ev[1], st));
  if (N < maxN && !c->p2p)
    CU_TRY(cudaMemsetAsync(c->topk + (size_t)N * k, 0xFF, sizeof(int) * (maxN - N) * k, st));
  // dispatch: every rank's tokens and routing to every rank (fixed counts, no host sync)
  const int nY = (H + 511) / 512;
  if (c->p2p) {
    // dispatched by the route kernel above (route.cuh, ep_P > 0)
  } else {
    const ncclDataType_t xt = c->bf16 ? ncclBfloat16 : ncclFloat32;
    NC_TRY(ncclGroupStart());
    NC_TRY(ncclAllGather(c->x_in, c->x_all, (size_t)maxN * H, xt, c->comm, st));
    NC_TRY(ncclAllGather(c->topk, c->topk_all, (size_t)maxN * k, ncclInt32, c->comm, st));
    NC_TRY(ncclAllGather(c->gates, c->gates_all, (size_t)maxN * k, ncclFloat32, c->comm, st));
    NC_TRY(ncclGroupEnd());
  }
  if (c->timing) CU_TRY(cudaEventRecord(rec.ev[2], st));
  // local experts' token lists over all rows; their counts are the global hits (R-18)
  if (c->p2p) {
    // built by the route grid's last CTA once every rank dispatched (route_ep_lists)
  } else {
    CU_TRY(cudaMemsetAsync(c->cnt_l, 0, sizeof(int) * El, st));
    tide_ep_lists_kernel<<<(R * k + 255) / 256, 256, 0, st>>>(c->topk_all, R, k, c->e0, El,
                                                            c->cnt_l, c->list_l, R, c->pslot_all);
    CU_TRY(cudaGetLastError());
    c->launches++;
  }
  // a4: placement of the local experts runs beside the FFN on the side stream (the FFN
  // computes every hit local expert; placement' only drives I/O), joined before the end
  CU_TRY(cudaEventRecord(c->ev_route, st));
  CU_TRY(cudaStreamWaitEvent(c->side, c->ev_route, 0));
  s = launch_book(c, c->cnt_l, placement, 0, refresh, capacity, c->hits_l, placement_out, c->side,
                  El, step, c->p2p ? c->cnt_par : nullptr);  // p2p: [2][El] by parity
  if (s != TIDE_OK) return s;
  CU_TRY(cudaEventRecord(c->ev_book, c->side));
  if (c->timing) CU_TRY(cudaEventRecord(rec.ev[3], st));
  // a7: grouped FFN over the local experts (+ shared expert on this rank's tokens)
  s = launch_ffn(c, c->cnt_l, nullptr, nullptr, nullptr, c->ffn_ctrl, c->ffn_ctrl + 1, N, st, true,
                 nullptr, c->p2p ? c->cnt_par : nullptr,
                 /*prefetch: the next layer's local experts into L2*/ true);
  if (s != TIDE_OK) return s;
  if (c->timing) CU_TRY(cudaEventRecord(rec.ev[4], st));
  // a10: per-source partial sums, exchange, rank-order sum
  const int srow = shared ? R * k : -1;
  if (c->p2p) {  // the FFN stored every pair's y at its owner and arrived (ffn.cuh)
    if (c->timing) CU_TRY(cudaEventRecord(rec.ev[5], st));
    CU_TRY(cudaStreamWaitEvent(st, c->ev_book, 0));  // a4 joined before the last kernel (see tide_moe_step)
    const dim3 grid(std::max(N, 1), nY);
    // one arrival per FFN CTA of every rank; none at world 1 (stream order suffices)
    const unsigned tgt = c->world > 1 ? (unsigned)c->ep_arrivals : 0u;
    if (c->bf16)
      CU_TRY(launch_pdl(tide_ep_final_p2p_kernel<__nv_bfloat16>, grid, dim3(128), 0, st, c->sym,
                        c->lay, (const int*)c->cnt_par, tgt, (const float*)c->gates,
                        (const float*)c->y_perm, static_cast<__nv_bfloat16*>(out), hit_counts,
                        c->E, N, k, H, srow));
    else
      CU_TRY(launch_pdl(tide_ep_final_p2p_kernel<float>, grid, dim3(128), 0, st, c->sym, c->lay,
                        (const int*)c->cnt_par, tgt, (const float*)c->gates,
                        (const float*)c->y_perm, static_cast<float*>(out), hit_counts, c->E, N,
                        k, H, srow));
    c->launches++;
  } else {
    CU_TRY(launch_pdl(tide_ep_partial_kernel, dim3(R, nY), dim3(128), 0, st,
                      (const float*)c->y_perm, (const int*)c->topk_all, (const float*)c->gates_all,
                      (const int*)c->pslot_all, (const int*)c->off_l, c->partial, k, H, c->e0, El));
    c->launches++;
    NC_TRY(ncclAlltoAll(c->partial, c->recv, (size_t)maxN * H, ncclFloat32, c->comm, st));
    if (c->timing) CU_TRY(cudaEventRecord(rec.ev[5], st));
    if (N > 0) {
      const dim3 grid(N, nY);
      if (c->bf16)
        CU_TRY(launch_pdl(tide_ep_final_kernel<__nv_bfloat16>, grid, dim3(128), 0, st,
                          (const float*)c->recv, (const float*)c->y_perm,
                          static_cast<__nv_bfloat16*>(out), c->world, maxN, H, srow));
      else
        CU_TRY(launch_pdl(tide_ep_final_kernel<float>, grid, dim3(128), 0, st, (const float*)c->recv,
                          (const float*)c->y_perm, static_cast<float*>(out), c->world, maxN, H,
                          srow));
      c->launches++;
    }
    NC_TRY(ncclAllGather(c->cnt_l, hit_counts, (size_t)El, ncclInt32, c->comm, st));
  }
  if (!c->p2p) CU_TRY(cudaStreamWaitEvent(st, c->ev_book, 0));  // placement_out / info valid with the stream
  if (!c->ev_ep_done) CU_TRY(cudaEventCreateWithFlags(&c->ev_ep_done, cudaEventDisableTiming));
  CU_TRY(cudaEventRecord(c->ev_ep_done, st));  // tide_ctx_ep_wait
  if (c->timing) {
    CU_TRY(cudaEventRecord(rec.ev[6], st));
    rec.launches = c->launches - launches0;
    rec.ffn_launches = c->ffn_launches - ffn0;
    c->pending.push_back(rec);
  }
  if (stats) {
    RouteInfo local;
    std::vector<int> hl(El);
    CU_TRY(cudaMemcpyAsync(&local, c->info, sizeof(RouteInfo), cudaMemcpyDeviceToHost, st));
    CU_TRY(cudaMemcpyAsync(hl.data(), c->hits_l, sizeof(int) * El, cudaMemcpyDeviceToHost, st));
    CU_TRY(cudaStreamSynchronize(st));
    if (local.status != 0)
      return fail(TIDE_EPLACEMENT, "step %d is not a refresh and placement holds more than %d experts",
                  step, capacity);
    int64_t wb = 0;
    for (int e = 0; e < El; ++e) wb += (int64_t)c->expert_bytes * ((hl[e] + kMaxTok - 1) / kMaxTok);
    if (shared) wb += (int64_t)c->expert_bytes * ((N + kMaxTok - 1) / kMaxTok);
    int pairs_l = 0;
    for (int e = 0; e < El; ++e) pairs_l += hl[e];
    fill_stats(c, &local, N, 0, 0, wb, stats, wb, pairs_l + (shared ? N : 0), 1);
    stats->nonresident_pairs = 0;
    for (int e = 0; e < El; ++e) stats->nonresident_pairs += hl[e];
    stats->nonresident_pairs -= local.resident_pairs;
  }
  return TIDE_OK;
}

// ---------------------------------------------------------------- NEXT-2 (host)
tide_status tide_interval_cost(const tide_interval_model* m, int32_t tau, double* io_cost,
                               double* miss_cost) {
  if (!m || !io_cost || !miss_cost) return fail(TIDE_EINVAL, "null argument");
  if (tau < 1 || m->B < 1 || m->T < 1 || m->d < 0.0 || m->d > 1.0)
    return fail(TIDE_EINVAL, "tau %d / B %d / T %d / d %g out of range", tau, m->B, m->T, m->d);
  // Eq. 5: c_io * (B*T/tau) * (1 - (1-d)^tau)
  double keep = 1.0;
  for (int j = 0; j < tau; ++j) keep *= 1.0 - m->d;
  *io_cost = m->c_io * ((double)m->B * m->T / tau) * (1.0 - keep);
  // Eq. 6: c_miss * T * B * f(tau), f = mean stale fraction (1/tau) sum_{j<tau} (1-(1-d)^j)
  double f = 0.0, kj = 1.0;
  for (int j = 0; j < tau; ++j) {
    f += 1.0 - kj;
    kj *= 1.0 - m->d;
  }
  *miss_cost = m->c_miss * (double)m->T * m->B * (f / tau);
  return TIDE_OK;
}

tide_status tide_optimize_interval(const tide_interval_model* m, int32_t* tau_out, double* curve) {
  if (!m || !tau_out) return fail(TIDE_EINVAL, "null argument");
  if (m->T < 2) return fail(TIDE_EINVAL, "T %d < 2", m->T);
  int best = 1;
  double best_c = 0.0;
  for (int tau = 1; tau <= m->T - 1; ++tau) {  // Eq. 7 domain, exhaustive
    double io, ms;
    tide_status s = tide_interval_cost(m, tau, &io, &ms);
    if (s != TIDE_OK) return s;
    if (curve) curve[tau - 1] = io + ms;
    if (tau == 1 || io + ms < best_c) {
      best = tau;
      best_c = io + ms;
    }
  }
  *tau_out = best;
  return TIDE_OK;
}

// NEXT-2 on B200: expert copies of a refresh interval measured on a routing trace.
tide_status tide_interval_profile(const int32_t* counts, int32_t T, int32_t E, int32_t B,
                                  double* miss_lag, double* mig_lag) {
  if (!counts || !miss_lag || !mig_lag) return fail(TIDE_EINVAL, "null argument");
  if (T < 1 || E < 1 || B < 1 || B > E) return fail(TIDE_EINVAL, "T %d / E %d / B %d", T, E, B);
  // top-B of every step by (hits desc, id asc): the placement rule (R-8)
  std::vector<uint8_t> top((size_t)T * E, 0);
  std::vector<int> ids(E);
  for (int t = 0; t < T; ++t) {
    const int32_t* c = counts + (size_t)t * E;
    for (int e = 0; e < E; ++e) ids[e] = e;
    std::stable_sort(ids.begin(), ids.end(), [c](int a, int b) { return c[a] > c[b]; });
    for (int i = 0; i < B; ++i) top[(size_t)t * E + ids[i]] = 1;
  }
  for (int j = 0; j < T; ++j) {
    int64_t miss = 0, mig = 0;
    for (int t = 0; t + j < T; ++t) {
      const uint8_t* r = &top[(size_t)t * E];
      const uint8_t* r2 = &top[(size_t)(t + j) * E];
      const int32_t* c2 = counts + (size_t)(t + j) * E;
      for (int e = 0; e < E; ++e) {
        miss += (c2[e] > 0 && !r[e]);
        mig += (r2[e] && !r[e]);
      }
    }
    miss_lag[j] = (double)miss / (double)(T - j);
    mig_lag[j] = (double)mig / (double)(T - j);
  }
  return TIDE_OK;
}

tide_status tide_interval_cost_trace(const tide_interval_trace_model* m, int32_t tau,
                                     double* copies, double* cost) {
  if (!m || !m->miss_lag || !m->mig_lag || !copies || !cost) return fail(TIDE_EINVAL, "null argument");
  if (tau < 1 || tau >= m->T) return fail(TIDE_EINVAL, "tau %d outside [1, T-1 = %d]", tau, m->T - 1);
  double per = m->mig_lag[tau];  // one interval: the refresh's promotions + tau steps of misses
  for (int j = 0; j < tau; ++j) per += m->miss_lag[j];
  *copies = (double)m->T / (double)tau * per;
  *cost = m->c_io * *copies + (double)m->T * m->c_step;
  return TIDE_OK;
}

tide_status tide_optimize_interval_trace(const tide_interval_trace_model* m, int32_t* tau_out,
                                         double* curve) {
  if (!m || !tau_out) return fail(TIDE_EINVAL, "null argument");
  if (m->T < 2) return fail(TIDE_EINVAL, "T %d < 2", m->T);
  int best = 1;
  double best_c = 0.0;
  for (int tau = 1; tau <= m->T - 1; ++tau) {  // Eq. 7 domain, exhaustive
    double cp, c;
    tide_status s = tide_interval_cost_trace(m, tau, &cp, &c);
    if (s != TIDE_OK) return s;
    if (curve) curve[tau - 1] = c;
    if (tau == 1 || c < best_c) {
      best = tau;
      best_c = c;
    }
  }
  *tau_out = best;
  return TIDE_OK;
}

// NEXT-2 replay (R-24): the host_master step's placement and copy rules over a trace.
tide_status tide_interval_replay(const int32_t* counts, int32_t T, int32_t E, int32_t B,
                                 int32_t tau, int32_t lazy, int32_t passes, int64_t* copies,
                                 int32_t* copies_per_step) {
  if (!counts || !copies) return fail(TIDE_EINVAL, "null argument");
  if (T < 1 || E < 1 || B < 1 || B > E || tau < 1 || passes < 1)
    return fail(TIDE_EINVAL, "T %d / E %d / B %d / tau %d / passes %d", T, E, B, tau, passes);
  std::vector<uint8_t> placed(E, 0), in_hbm(E, 0);
  std::vector<int> ids(E);
  int64_t total = 0;
  for (int pass = 0; pass < passes; ++pass)
    for (int t = 0; t < T; ++t) {
      const int32_t* c = counts + (size_t)t * E;
      if (t % tau == 0) {  // refresh: top-B by (hits desc, id asc)
        for (int e = 0; e < E; ++e) ids[e] = e;
        std::stable_sort(ids.begin(), ids.end(), [c](int a, int b) { return c[a] > c[b]; });
        std::fill(placed.begin(), placed.end(), 0);
        for (int i = 0; i < B; ++i) placed[ids[i]] = 1;
      }
      int n = 0;
      for (int e = 0; e < E; ++e) {
        if (in_hbm[e]) {  // served from its slot; an evicted slot is freed after the step
          in_hbm[e] = placed[e];
        } else if (placed[e] && (c[e] > 0 || !lazy)) {  // promoted: copied into its slot
          ++n;
          in_hbm[e] = 1;
        } else if (c[e] > 0) {  // streamed through staging for this step only
          ++n;
        }
      }
      if (pass == passes - 1) {
        total += n;
        if (copies_per_step) copies_per_step[t] = n;
      }
    }
  *copies = total;
  return TIDE_OK;
}

tide_status tide_optimize_interval_replay(const tide_interval_replay_model* m, int32_t tau_max,
                                          int32_t* tau_out, double* curve) {
  if (!m || !tau_out) return fail(TIDE_EINVAL, "null argument");
  if (tau_max < 1) return fail(TIDE_EINVAL, "tau_max %d < 1", tau_max);
  int best = 1;
  double best_c = 0.0;
  for (int tau = 1; tau <= tau_max; ++tau) {  // Eq. 7, exhaustive
    int64_t cp = 0;
    tide_status s = tide_interval_replay(m->counts, m->T, m->E, m->B, tau, m->lazy, m->passes,
                                         &cp, nullptr);
    if (s != TIDE_OK) return s;
    const double c = m->c_io * (double)cp + (double)m->T * m->c_step;
    if (curve) curve[tau - 1] = c;
    if (tau == 1 || c < best_c) {
      best = tau;
      best_c = c;
    }
  }
  *tau_out = best;
  return TIDE_OK;
}

// ---------------------------------------------------------------- NEXT-4 (device)
tide_status tide_trace_stats(const int32_t* counts, int32_t T, int32_t E, int32_t B, double* sim,
                             int32_t* unique, double* drift, void* stream) {
  if (!counts || !sim || !unique || !drift) return fail(TIDE_EINVAL, "null argument");
  if (T < 1 || E < 1 || E > 4096 || B < 1 || B > E) return fail(TIDE_EINVAL, "bad T/E/B");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  tide_trace_sim_kernel<<<dim3(T, T), 256, 0, st>>>(counts, T, E, sim);
  CU_TRY(cudaGetLastError());
  tide_trace_step_kernel<<<T, 1024, 2 * E, st>>>(counts, T, E, B, unique, drift);
  CU_TRY(cudaGetLastError());
  return TIDE_OK;
}

tide_status tide_ctx_set_prefetch(tide_ctx* c, tide_ctx* next, const void* next_device_all,
                                  int64_t budget_bytes) {
  if (!c) return fail(TIDE_EINVAL, "null context");
  if (budget_bytes < 0) return fail(TIDE_EINVAL, "budget_bytes %lld < 0", (long long)budget_bytes);
  if (next && next->device != c->device)
    return fail(TIDE_EINVAL, "next context is on device %d, this one on %d", next->device, c->device);
  if (next && !next_device_all) {  // host_master: H2D prefetch into `next`'s prefetch slots
    if (next->pool && next->pf_slots_req == 0)
      return fail(TIDE_EINVAL, "H2D prefetch for a context that already ran a host_master step");
    if (!next->pool)
      next->pf_slots_req = (int)std::min<int64_t>(std::min(next->E, 64),
                                                  budget_bytes / (int64_t)next->expert_bytes);
    c->pf_next_h = next->pf_slots_req > 0 ? next : nullptr;
    c->pf_next = nullptr;
    c->pf_weights = nullptr;
    c->pf_max = 0;
    return TIDE_OK;
  }
  if (c->pf_next) c->pf_next->pf_prev_budget = 0;
  if (!next || budget_bytes == 0) {
    c->pf_next = nullptr;
    c->pf_weights = nullptr;
    c->pf_max = 0;
    c->pf_next_h = nullptr;
    return TIDE_OK;
  }
  c->pf_next = next;
  c->pf_weights = next_device_all;
  c->pf_max = (int)std::min<int64_t>(next->E, budget_bytes / (int64_t)next->expert_bytes);
  c->pf_budget = budget_bytes;
  next->pf_target = true;
  next->pf_prev_budget = budget_bytes;
  return TIDE_OK;
}

tide_status tide_ctx_set_timing(tide_ctx* c, int32_t enable) {
  if (!c) return fail(TIDE_EINVAL, "ctx is null");
  tide_phase_times t;
  tide_status s = tide_ctx_get_timing(c, &t);  // drain
  if (s != TIDE_OK) return s;
  c->acc = tide_phase_times{};
  c->timing = enable != 0;
  return TIDE_OK;
}

tide_status tide_ctx_get_timing(tide_ctx* c, tide_phase_times* out) {
  if (!c || !out) return fail(TIDE_EINVAL, "null argument");
  CU_TRY(cudaSetDevice(c->device));
  for (auto& r : c->pending) {
    CU_TRY(cudaEventSynchronize(r.ev[6]));
    float ms[6];
    for (int i = 0; i < 6; ++i) CU_TRY(cudaEventElapsedTime(&ms[i], r.ev[i], r.ev[i + 1]));
    c->acc.router_ms += ms[0];
    c->acc.route_ms += ms[1];
    c->acc.gather_ms += ms[2];
    c->acc.ffn_ms += ms[3];
    c->acc.staged_ms += ms[4];
    c->acc.combine_ms += ms[5];
    float tot;
    CU_TRY(cudaEventElapsedTime(&tot, r.ev[0], r.ev[6]));
    c->acc.total_ms += tot;
    c->acc.steps += 1;
    c->acc.launches += r.launches;
    c->acc.ffn_launches += r.ffn_launches;
    for (cudaEvent_t e : r.ev) c->ev_pool.push_back(e);
  }
  c->pending.clear();
  *out = c->acc;
  return TIDE_OK;
}

}  // extern "C"
