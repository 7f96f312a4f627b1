/*
 * tide.h -- C ABI of the B200-native TIDE MoE layer-step (arXiv 2605.20179).
 *
 * One call, tide_moe_step(), runs one MoE layer at one denoising step for all
 * tokens of the block(s) at once (Alg. 1):
 *
 *   a1 router logits        l = X Wr^T
 *   a2 softmax + top-k      lowest id wins ties             (R-1..R-4)
 *   a3 hit histogram        hits[e] = #{(n,j): topk = e}
 *   a4 refresh + placement  if step % interval == 0:
 *                           top-`capacity` experts by hits
 *   a5 buckets              resident first, ascending id    (R-11)
 *   a6 non-resident I/O     pinned host -> HBM, side stream (R-13)
 *   a7/a8 grouped SwiGLU    y = Wd (silu(Wg x) * Wu x)      (north_star)
 *   a9 shared expert        (flag)                          (R-16)
 *   a10 combine             out[n] = sum_j g[n,j] y[n,j]
 *
 * P:n = /root/reference/PAPER.md line n; R-x = a reading in DESIGN.md section 3.
 *
 * Conventions
 *  - Every pointer is owned by the caller unless stated otherwise.  "device"
 *    pointers are CUDA device (HBM) addresses on the context's device; "host"
 *    pointers are CPU addresses.
 *  - `stream` is a cudaStream_t passed as void*; all device work of a call is
 *    ordered on it and outputs are valid once it completes.
 *  - Every entry point returns tide_status; no C++ exception crosses the ABI.
 *    tide_last_error() returns a thread-local message for the last failure.
 *  - Argument checks run before any work is enqueued; on TIDE_EINVAL /
 *    TIDE_ECAPACITY / TIDE_EUNSUPPORTED nothing was enqueued.  The one
 *    exception is TIDE_EPLACEMENT (see tide_moe_step).
 *  - Asynchronous device faults surface as TIDE_ECUDA at a later call.
 */
#ifndef TIDE_H
#define TIDE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TIDE_ABI_VERSION 2

#if defined(__GNUC__)
#define TIDE_API __attribute__((visibility("default")))
#else
#define TIDE_API
#endif

typedef enum {
  TIDE_OK = 0,
  TIDE_EINVAL = 1,        /* bad argument (null pointer, size out of range)        */
  TIDE_ECAPACITY = 2,     /* capacity outside [1, E] (or [1, E/P] under EP)        */
  TIDE_EPLACEMENT = 3,    /* non-refresh step with popcount(placement) > capacity */
  TIDE_ECUDA = 4,         /* CUDA runtime/driver failure                           */
  TIDE_ENCCL = 5,         /* NCCL failure (EP)                                     */
  TIDE_ENOMEM = 6,        /* device or pinned allocation failed                    */
  TIDE_EUNSUPPORTED = 7   /* shape/flag combination this build does not support    */
} tide_status;

/* Element type of activations, router weights, expert weights and `out`.   */
typedef enum { TIDE_F32 = 0, TIDE_BF16 = 1 } tide_dtype;

enum {
  TIDE_NORM_TOPK = 1u << 0,     /* renormalise the k selected gates (R-2)          */
  TIDE_SHARED_EXPERT = 1u << 1, /* add one always-resident shared expert (R-16)    */
  TIDE_LAZY_PROMOTE = 1u << 2,  /* copy a promoted expert on its first hit (R-9)   */
  /* NEXT-1 hit-counter readings (default: the current step's hits, R-5).  With one of
   * these, a refresh ranks experts by hits accumulated over earlier steps of the block
   * (no lookahead): WINDOW = since the previous refresh, reset at each refresh (SPEC
   * S:242); CUMULATIVE = since the block's step 0.  Step 0 ranks by its own hits. */
  TIDE_COUNTER_WINDOW = 1u << 3,
  TIDE_COUNTER_CUMULATIVE = 1u << 4,
  TIDE_TIE_INCUMBENT = 1u << 5  /* equal counts: experts already resident rank first */
};

/* Shape of one MoE layer.  Constraints checked by tide_ctx_create:
 *   1 <= top_k <= num_experts <= 1024, hidden and ffn multiples of 64,
 *   64 <= hidden <= 16384, 64 <= ffn <= 16384, 1 <= max_tokens <= 1024.     */
typedef struct {
  int32_t num_experts; /* E                                                   */
  int32_t top_k;       /* k                                                   */
  int32_t hidden;      /* model width H                                       */
  int32_t ffn;         /* expert intermediate width F (shared expert too)     */
  int32_t max_tokens;  /* largest num_tokens a step will be called with        */
  tide_dtype dtype;    /* TIDE_BF16 (tcgen05 kind::f16) or TIDE_F32 (kind::tf32) */
  uint32_t flags;      /* TIDE_NORM_TOPK | TIDE_SHARED_EXPERT | TIDE_LAZY_PROMOTE */
} tide_layer_desc;

/* Packed expert layout ("pack"): one expert = [Wg (F x H); Wu (F x H); Wd (H x F)],
 * each row-major, contiguous, 3*H*F elements of `dtype`.  Wg/Wu rows are the
 * F gate/up projections of the hidden vector, Wd rows the H outputs.      */
TIDE_API size_t tide_expert_elems(const tide_layer_desc* desc);
TIDE_API size_t tide_expert_bytes(const tide_layer_desc* desc);

/* Copy one expert's three matrices into packed form at `dst`.  Any of the
 * pointers may be host or device (unified addressing); the copy is enqueued
 * on `stream` (cudaMemcpyAsync, cudaMemcpyDefault).                        */
TIDE_API tide_status tide_pack_expert(const tide_layer_desc* desc, const void* w_gate, const void* w_up,
                             const void* w_down, void* dst, void* stream);

/* Where the experts' weights live.  Exactly one of device_all / host_master
 * must be non-NULL.
 *  device_all : device, E packed experts back to back (no offload: every expert
 *               is served from HBM; placement is still computed and reported).
 *  host_master: host, E packed experts back to back, PINNED (cudaHostAlloc or
 *               cudaHostRegister; checked, else TIDE_EINVAL).  Experts are
 *               copied into the context's HBM slot pool (capacity slots) and
 *               staging ring (see tide_ctx_create) as placement and hits demand.
 *               Must stay valid and unchanged for the lifetime of the context.
 *  shared_w   : device, one packed expert; required iff TIDE_SHARED_EXPERT.   */
typedef struct {
  const void* device_all;
  const void* host_master;
  const void* shared_w;
} tide_expert_weights;

/* Per-step counters (host struct, filled when `stats` is non-NULL; filling it
 * synchronises `stream`).                                                  */
typedef struct {
  int32_t refreshed;          /* step % interval == 0                                    */
  int32_t resident_pairs;     /* (token, expert) pairs whose expert is in placement'     */
  int32_t nonresident_pairs;  /* N*k - resident_pairs                                    */
  int32_t promotions;         /* |placement' \ placement|                                */
  int32_t evictions;          /* |placement \ placement'|                                */
  int32_t unique_experts;     /* experts with hits > 0                                   */
  int32_t experts_streamed;   /* hit experts whose weights were not in HBM at step start */
  int32_t copies;             /* expert H2D copies enqueued this step (incl. eager promotions) */
  int64_t h2d_bytes;          /* copies * tide_expert_bytes                              */
  int64_t weight_bytes_read;  /* expert weight bytes the grouped FFN streamed from HBM   */
  /* the first FFN launch of the step (experts whose weights were in HBM at step start,
   * + the shared expert); host_master mode runs one more launch per staged chunk      */
  int64_t resident_weight_bytes; /* weight bytes that launch streamed                  */
  int32_t resident_rows;      /* token rows it computed (routed pairs + shared rows)     */
  int32_t ffn_launches;       /* grouped-FFN launches of this step                       */
} tide_step_stats;

/* Optional device outputs for tests (nullable members, device pointers).  */
typedef struct {
  int32_t* topk_idx; /* [N, k] ranked expert ids                                  */
  float* gates;      /* [N, k]                                                    */
  int32_t* pos;      /* [N, k] row of pair (n, j) in bucket order (R-11)          */
  int32_t* order;    /* [E] expert at each bucket position                        */
  int32_t* offsets;  /* [E + 1] first row of each bucket position                 */
  float* logits;     /* [N, E] fp32 router logits                                 */
  uint64_t* route_trace; /* [8 * route CTAs] %globaltimer ns per route-kernel CTA:
                            start, phase 1 done, phase 2 start, phase 2 done, then (phase-2
                            CTAs, warp 0) logits loaded, selection done, histogram done
                            (0 = n/a); needs >= 8 * ceil(E/8) * ceil(N/4) entries       */
  uint64_t* ffn_trace;   /* [8 * #SMs] per FFN CTA: entry, work list ready, producer done,
                            epilogue done (%globaltimer ns), items processed                */
  uint64_t* ffn_item_trace; /* [4 * 64 * #SMs] per FFN CTA, its first 64 items: claim time,
                            kind << 32 | entry, dependency met, last load issued (ns)      */
} tide_step_debug;

typedef struct tide_ctx tide_ctx;

/* Create a context for one layer on `device`.
 *  capacity      : C, HBM-resident experts for this layer (1 <= C <= E).  In
 *                  host_master mode the context owns C HBM slots.
 *  staging_slots : S >= 2, HBM staging ring for non-resident hits (R-13); the
 *                  ring is allocated on the first host_master step (S * expert
 *                  bytes) and is reported as HBM overhead beyond C.
 * The context owns its workspaces (sized by max_tokens), slot pool, staging
 * ring, streams and events.  Not thread-safe; distinct contexts may run
 * concurrently on distinct streams.                                         */
TIDE_API tide_status tide_ctx_create(const tide_layer_desc* desc, int32_t capacity, int32_t staging_slots,
                            int32_t device, tide_ctx** out);
TIDE_API void tide_ctx_destroy(tide_ctx* ctx);

/* One MoE layer-step.
 *  block_hidden  : device [num_tokens, H] of dtype, the block's hidden states.
 *  num_tokens    : N, 0 <= N <= max_tokens.
 *  router_w      : device [E, H] of dtype.
 *  expert_w      : weights, see tide_expert_weights.
 *  placement     : device [E] uint8, nonzero = resident (the caller's current
 *                  placement; at step 0 of a block any value, R-7).
 *  step          : denoising step within the block, >= 0.
 *  interval      : refresh interval tau >= 1; refresh iff step % interval == 0.
 *  capacity      : must equal the context's capacity.
 *  out           : device [N, H] of dtype.
 *  hit_counts    : device [E] int32, this step's hits (Sum = N*k).
 *  placement_out : device [E] uint8, placement' (may alias `placement`).
 * Returns TIDE_EPLACEMENT when the step is not a refresh and the input
 * placement holds more than `capacity` experts.  That check runs on the
 * device, in the bookkeeping kernel after the router: when it fails,
 * hit_counts holds this step's hits, placement_out is a copy of the input
 * placement (unchanged), and no bucket / pos / I/O work is done.  In
 * device_all mode the FFN and combine still run (they compute every hit
 * expert whatever the placement, so `out` holds the layer's output); in
 * host_master mode the resident FFN has run, no H2D copy or staged FFN is
 * enqueued and `out` is not valid.  In device_all mode (no offload) the
 * status is reported only when `stats` is requested (the call does not
 * otherwise synchronise); host_master mode always reports it.
 * In host_master mode the call blocks once on an internal event after the
 * routing kernels to read the <= E-entry miss list, then enqueues H2D copies
 * on an internal side stream, overlapped with the resident experts' FFN.   */
TIDE_API tide_status tide_moe_step(tide_ctx* ctx, const void* block_hidden, int32_t num_tokens,
                          const void* router_w, const tide_expert_weights* expert_w,
                          const uint8_t* placement, int32_t step, int32_t interval,
                          int32_t capacity, void* out, int32_t* hit_counts,
                          uint8_t* placement_out, tide_step_stats* stats, tide_step_debug* dbg,
                          void* stream);

/* ------------------------------------------------------------------------
 * Expert parallelism (DESIGN R-18), one process per GPU.
 * Rank r of P owns experts [r*E/P, (r+1)*E/P); each rank routes its own tokens.
 * A step: route (local tokens) -> ncclAllGather of tokens, top-k ids and gates
 * (fixed max_tokens rows per rank, no host sync) -> grouped FFN over the local
 * experts for every rank's tokens -> per-source partial sums (fp32, slot order)
 * -> ncclAlltoAll -> out = sum of the P partials in rank order (+ shared expert).
 * hit_counts is global ([E], ncclAllGather of the local experts' counts);
 * placement / placement_out cover the rank's E/P local experts (device [E/P]);
 * capacity is per rank (1 <= C <= E/P).  The context owns its NCCL communicator.
 * ------------------------------------------------------------------------ */

/* Fill out[128] with a fresh ncclUniqueId (call on one rank, share the bytes). */
TIDE_API tide_status tide_nccl_unique_id(void* out);

/* Collective over the `world` ranks (each calls it with the same unique id).
 * E must be divisible by world. */
TIDE_API tide_status tide_ctx_create_ep(const tide_layer_desc* desc, int32_t device,
                                        const void* nccl_unique_id, int32_t rank, int32_t world,
                                        tide_ctx** out);

/* Another layer's context on the same rank/device sharing `parent`'s communicator
 * (parent must outlive it).  Not collective. */
TIDE_API tide_status tide_ctx_create_ep_like(const tide_layer_desc* desc, tide_ctx* parent,
                                             tide_ctx** out);

/* local_experts: device, E/P packed experts of this rank (expert r*E/P + i at slot i).
 * shared_w: device packed shared expert (iff TIDE_SHARED_EXPERT).  Other arguments as
 * tide_moe_step.  Every rank must call it for the same layer/step (collectives). */
TIDE_API tide_status tide_moe_step_ep(tide_ctx* ctx, const void* block_hidden, int32_t num_tokens,
                                      const void* router_w, const void* local_experts,
                                      const void* shared_w, const uint8_t* placement,
                                      int32_t step, int32_t interval, int32_t capacity, void* out,
                                      int32_t* hit_counts, uint8_t* placement_out,
                                      tide_step_stats* stats, void* stream);

/* ------------------------------------------------------------------------
 * Peer-memory expert parallelism (NEXT-3 "fused NVLink dispatch/combine", SURVEY 8(f);
 * the exchange of SURVEY 8(e) without NCCL on the data path).  Same step and arguments
 * as tide_moe_step_ep; the exchanges are done by the compute kernels themselves with
 * P2P stores into every rank's symmetric region (NVLink / NVSwitch):
 *  - dispatch fused into the router: each token row of X, its top-k ids, gates and the
 *    rank's token count go to every rank; one release arrival per source rank;
 *  - combine exchange fused into the grouped FFN: the tcgen05 epilogue stores each
 *    routed pair's y row into its token's rank; the FFN's last CTA delivers the local
 *    experts' hit counts and arrives once per rank (release, system scope);
 *  - the token's rank then runs the single-device combine (slot order, fp32, + shared
 *    expert), so out equals tide_moe_step's out bit for bit for every world size.
 * Consumers wait on the arrival counters with acquire loads (system scope).
 *
 * Setup, on every rank, per layer context:
 *   tide_ctx_create_ep_p2p(desc, device, rank, world, &ctx)    (world <= 8)
 *   tide_ctx_ep_export(ctx, handle, &base)   -> this rank's IPC handle
 *                                               (tide_ep_handle_bytes() bytes) and base
 *   exchange the handles (e.g. torch.distributed all_gather), then
 *   tide_ctx_ep_connect(ctx, handles, bases)  handles: world * handle_bytes in rank
 *                                               order; bases: nullable array of
 *                                               world pointers; a non-null entry is
 *                                               used as that peer's region directly
 *                                               (same process: single-GPU emulation)
 *   barrier across ranks before the first tide_moe_step_ep.
 * Ownership: the context owns its symmetric region and the peer mappings it opened
 * (closed by tide_ctx_destroy; destroy on every rank only after all ranks finished
 * their last step).  A waiting kernel gives up after 20 s, records the failure in the
 * context's error word (tide_ctx_ep_error) and returns without hanging the GPU; the
 * step's outputs are then undefined.  Not capturable across ranks' differing call
 * counts: every rank must call tide_moe_step_ep once per layer-step, in the same order.
 * ------------------------------------------------------------------------ */
TIDE_API tide_status tide_ctx_create_ep_p2p(const tide_layer_desc* desc, int32_t device,
                                            int32_t rank, int32_t world, tide_ctx** out);
TIDE_API size_t tide_ep_handle_bytes(void);
/* handle (nullable): out, tide_ep_handle_bytes() bytes; base (nullable): out, device ptr. */
TIDE_API tide_status tide_ctx_ep_export(tide_ctx* ctx, void* handle, void** base);
/* TIDE_EINVAL if not a peer-memory context, already connected, or a peer has neither a
 * handle nor a base; TIDE_ECUDA if cudaIpcOpenMemHandle fails. */
TIDE_API tide_status tide_ctx_ep_connect(tide_ctx* ctx, const void* handles,
                                         const void* const* bases);
/* *err = 1 if a peer-memory wait timed out since the context was created (synchronous). */
TIDE_API tide_status tide_ctx_ep_error(tide_ctx* ctx, int32_t* err);
/* Failure handling of an expert-parallel context (either exchange), host side: waits until
 * the context's last step has completed on the device, polling every ~50 us.  NCCL
 * contexts: an asynchronous communicator error (ncclCommGetAsyncError) or no completion
 * within `timeout_ms` aborts the communicator (ncclCommAbort: the collectives in flight
 * return, the context is unusable afterwards) and returns TIDE_ENCCL.  Peer-memory
 * contexts: a kernel-side wait that gave up (the error word) returns TIDE_ECUDA; no
 * completion within `timeout_ms` returns TIDE_ECUDA.  TIDE_OK when the step completed.  */
TIDE_API tide_status tide_ctx_ep_wait(tide_ctx* ctx, int32_t timeout_ms);

/* Per-phase device timing (CUDA events recorded on the step's stream at phase
 * boundaries).  Enabling resets the accumulators; tide_ctx_get_timing waits
 * for the recorded events, adds their elapsed times and clears them.
 *  router/route/gather/ffn/combine: a1, a2-a5, a5 gather, a7+a9 (experts in HBM),
 *  a10; staged: from the end of the resident FFN to the start of the combine
 *  in host_master mode (H2D waits + a8 FFN over staged chunks).
 *  launches: kernels this context launched while timing was enabled.
 *  Under EP (tide_moe_step_ep) the fields hold: router_ms = route kernel,
 *  route_ms = dispatch all-gather, gather_ms = local lists + placement, ffn_ms = FFN,
 *  staged_ms = partial sums + all-to-all, combine_ms = rank-order sum + hits gather.  */
typedef struct {
  double router_ms, route_ms, gather_ms, ffn_ms, staged_ms, combine_ms, total_ms;
  int64_t steps, launches, ffn_launches;
} tide_phase_times;
TIDE_API tide_status tide_ctx_set_timing(tide_ctx* ctx, int32_t enable);
TIDE_API tide_status tide_ctx_get_timing(tide_ctx* ctx, tide_phase_times* out);

/* ------------------------------------------------------------------------
 * NEXT-3: cross-layer L2 prefetch (P:278-281's "overlap" intent).
 * After this call, every device_all tide_moe_step on `ctx` ends its FFN by prefetching
 * into L2 (cp.async.bulk.prefetch.L2) the experts of `next` most likely to be hit at
 * next's coming step: the shared expert, then next's experts with hits > 0 at its most
 * recent step in ascending id (the order next's FFN claims them; TIDE_PF_BY_HITS=1 ranks
 * by hits instead), their gate/up rows (what the FFN's first items read) up to
 * budget_bytes. Each CTA of the persistent FFN issues its share once it has no more
 * work, so the prefetch fills the FFN tail, the combine and next's routing, when HBM
 * would otherwise be idle.  `next`'s own FFN then continues the same ranked list for
 * another budget_bytes / 2 (its persistent CTAs, resident while its routing is still being
 * computed, issue that share before they wait on the routing).
 *   next:            the context of the layer called after `ctx` (same device); NULL or
 *                    budget_bytes == 0 disables. `next` must outlive `ctx` or be unset.
 *   next_device_all: the packed experts `next` is called with ([E, 3HF], device), or
 *                    NULL when `next` serves its experts from a pinned host master
 *                    (host_master): then, at the end of every host_master step of `ctx`,
 *                    the experts next streamed at its previous step (hit, not in HBM;
 *                    most-hit first, up to budget_bytes / expert bytes, at most 64) are
 *                    copied host-to-HBM into `next`'s own prefetch slots on its side
 *                    stream, so the H2D link works through the gap before next's step
 *                    plans its copies; next's step computes those experts from the
 *                    prefetch slots (or moves a promoted one HBM-to-HBM) instead of
 *                    copying them again.  The slots are extra HBM owned by `next`; set this
 *                    before next's first host_master step.  Prefetch copies are counted in
 *                    next's stats (copies, h2d_bytes), wrong predictions included.
 * It is a cache / copy-timing hint only: outputs are bitwise unchanged. Nothing is
 * prefetched before `next` has run one step. Returns TIDE_EINVAL on a null ctx, negative
 * budget, different devices, or a host prefetch set after next's first host step.
 * ------------------------------------------------------------------------ */
TIDE_API tide_status tide_ctx_set_prefetch(tide_ctx* ctx, tide_ctx* next,
                                           const void* next_device_all, int64_t budget_bytes);

/* ------------------------------------------------------------------------
 * NEXT-2: refresh-interval model (Eq. 4-7), host-only.
 *   io(tau)   = c_io * (B*T/tau) * (1 - (1-d)^tau)                      (Eq. 5)
 *   miss(tau) = c_miss * T * B * f(tau), f(tau) = (1/tau) sum_{j<tau} (1-(1-d)^j)
 *                                                                        (Eq. 6)
 *   tau* = argmin over tau in [1, T-1] of io + miss, ties -> smallest     (Eq. 7)
 * d: drift rate (Eq. 4, e.g. from tide_trace_stats); c_io: cost of one expert
 * migration; c_miss: cost of one stale resident slot per step (on B200 the miss
 * is an H2D stream of the expert, R-13, so c_miss ~ c_io).  curve: [T-1] or NULL.
 * ------------------------------------------------------------------------ */
typedef struct {
  int32_t T, B;
  double d, c_io, c_miss;
} tide_interval_model;
TIDE_API tide_status tide_interval_cost(const tide_interval_model* m, int32_t tau,
                                        double* io_cost, double* miss_cost);
TIDE_API tide_status tide_optimize_interval(const tide_interval_model* m, int32_t* tau_out,
                                            double* curve);

/* NEXT-2 on B200 (DESIGN R-21): the same trade-off (Eq. 5 migrations vs Eq. 6 misses,
 * Eq. 7 scan) with the expert counts measured on a routing trace instead of derived from
 * a constant drift, and with the experts that stream at every step (hit but outside even
 * a fresh placement: R-13) included.  From host per-step hit counts [T][E]:
 *   miss_lag[j] = mean over t of |{e : counts[t+j][e] > 0} \ topB(counts[t])|
 *                 (hit experts outside a placement refreshed j steps earlier: streamed)
 *   mig_lag[j]  = mean over t of |topB(counts[t+j]) \ topB(counts[t])|
 *                 (promotions when a j-step-old placement is refreshed; Eq. 4 at lag j, x B)
 * for j = 0..T-1, means over t = 0..T-1-j; topB = the placement rule (hits desc, id asc,
 * R-8).  miss_lag / mig_lag: host [T].  1 <= B <= E, T >= 1.                            */
TIDE_API tide_status tide_interval_profile(const int32_t* counts, int32_t T, int32_t E, int32_t B,
                                           double* miss_lag, double* mig_lag);
/* Expert copies over a block of T steps when refreshing every tau steps (1 <= tau < T):
 *   copies(tau) = (T / tau) * (mig_lag[tau] + sum_{j < tau} miss_lag[j])
 * cost = c_io * copies + T * c_step (c_io: seconds per expert H2D copy; c_step: the
 * step's time without expert I/O).  tau* = argmin over [1, T-1], ties -> smallest tau;
 * curve: host [T-1] costs or NULL.                                                       */
typedef struct {
  int32_t T;
  double c_io, c_step;
  const double* miss_lag;  /* host [T] from tide_interval_profile */
  const double* mig_lag;   /* host [T] */
} tide_interval_trace_model;
TIDE_API tide_status tide_interval_cost_trace(const tide_interval_trace_model* m, int32_t tau,
                                              double* copies, double* cost);
TIDE_API tide_status tide_optimize_interval_trace(const tide_interval_trace_model* m,
                                                  int32_t* tau_out, double* curve);

/* NEXT-2 replay (DESIGN R-24): the exact expert copies of a refresh interval on a recorded
 * routing trace, instead of the stationary lag averages above.  Alg. 1 lines 3-4
 * are replayed step by step with the rules the library's own host_master step applies:
 * refresh iff t % tau == 0 within the block (a4), placement = top-B by (hits desc, id asc)
 * (R-5, R-8), copies: a hit expert not in HBM at the step's start is copied once (into its
 * slot if it is placed, else through staging: R-13), a placed expert with no hits is copied
 * at the refresh unless lazy (R-9), an evicted expert stays servable until the step ends
 * (R-12).  `passes` blocks of the same trace run back to back with the placement carried
 * across blocks (nothing in HBM before the first block); *copies is the total of the last
 * pass (passes >= 2: steady state), copies_per_step (host [T] or NULL) its per-step split.
 *  counts : host [T][E] int32 hit counts of one block (e.g. hit_counts of T steps)
 * Constraints: T >= 1, 1 <= B <= E, tau >= 1, passes >= 1; else TIDE_EINVAL.
 * NEXT-1 counter modes / incumbent ties are not replayed (mode 0 only).               */
TIDE_API tide_status tide_interval_replay(const int32_t* counts, int32_t T, int32_t E, int32_t B,
                                          int32_t tau, int32_t lazy, int32_t passes,
                                          int64_t* copies, int32_t* copies_per_step);
/* Eq. 7 over the replay: cost(tau) = c_io * copies(tau) + T * c_step for tau = 1..tau_max
 * (exhaustive, ties -> smallest tau); curve: host [tau_max] costs or NULL.             */
typedef struct {
  const int32_t* counts;  /* host [T][E] */
  int32_t T, E, B, lazy, passes;
  double c_io, c_step;
} tide_interval_replay_model;
TIDE_API tide_status tide_optimize_interval_replay(const tide_interval_replay_model* m,
                                                   int32_t tau_max, int32_t* tau_out,
                                                   double* curve);

/* NEXT-4: routing-trace analytics on the device.
 *  counts : device [T][E] int32 per-step hit counts (e.g. hit_counts of T steps)
 *  sim    : device [T][T] fp64 cosine similarity of the count vectors (0 if a vector is 0)
 *  unique : device [T] experts with hits > 0 per step
 *  drift  : device [T-1] Eq. 4 drift of the top-B placement between consecutive steps
 * Enqueued on `stream`; 1 <= B <= E <= 4096. */
TIDE_API tide_status tide_trace_stats(const int32_t* counts, int32_t T, int32_t E, int32_t B,
                                      double* sim, int32_t* unique, double* drift,
                                      void* stream);

/* Thread-local description of the last failure on this thread. */
TIDE_API const char* tide_last_error(void);

/* ABI version (TIDE_ABI_VERSION) and the device kernels' SM target (100). */
TIDE_API int32_t tide_abi_version(void);
TIDE_API int32_t tide_build_sm(void);

#ifdef __cplusplus
}
#endif
#endif /* TIDE_H */
