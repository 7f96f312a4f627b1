/*
 * tide_oracle.h -- plain CPU reference ("oracle") of one TIDE MoE layer-step.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (libtide.so, paper_2605_20179_b200/) never links, imports
 * or calls it, and it shares no code, header, table or helper with the CUDA
 * path.  See oracle/tide_oracle.c for the per-function paper citations.
 *
 * Citation keys: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n,
 * "DESIGN R-x" = a reading listed in DESIGN.md section "Readings".
 *
 * All floating point is fp64.  Inputs are the stored bytes (fp32 or bf16
 * bit patterns), converted exactly to double on read.
 */
#ifndef TIDE_ORACLE_H
#define TIDE_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_F32 = 0, ORC_BF16 = 1 };

/* Host threads for the per-token loops (OpenMP).  Results are bit-identical for any
 * count: a token's arithmetic never crosses threads.                                */
void orc_set_threads(int n);
int orc_get_threads(void);

/* O1: logits[n*E+e] = sum_h x[n,h]*wr[e,h], summed in h order. */
int orc_router_logits(int N, int E, int hidden, const void* x, int x_dtype,
                      const void* wr, int wr_dtype, double* logits);

/* O2: per token, the k largest logits, ties -> lower id.
 * topk_idx[n*k+j] is the j-th ranked expert.  Stable selection.       */
int orc_topk(int N, int E, int k, const double* logits, int32_t* topk_idx);

/* O3: gates.  norm_topk=1: g = p_e / sum_{selected} p (DESIGN R-2);
 * norm_topk=0: g = p_e, p = softmax over all E logits.                 */
int orc_gates(int N, int E, int k, const double* logits, const int32_t* topk_idx,
              int norm_topk, double* gates);

/* O4 (Alg.1 H): hits[e] = #{(n,j): topk_idx[n,j] == e}.            */
int orc_hits(int N, int E, int k, const int32_t* topk_idx, int32_t* hits);

/* O5 (Alg.1 line 2): refresh iff step % interval == 0.           */
int orc_is_refresh(int step, int interval);

/* O6 (DESIGN R-6/R-8): at a refresh the resident set
 * is the top-C experts by (hits desc, id asc); otherwise the input set.   */
int orc_placement(int E, int capacity, const int32_t* hits, int refresh,
                  const uint8_t* placement_in, uint8_t* placement_out);

/* O7 (DESIGN R-11): bucket order = resident ascending id, then
 * non-resident ascending id.  order[i] = expert at bucket position i,
 * offsets[i] = first row of order[i] (offsets[E] = N*k),
 * pos[n*k+j] = row of pair (n,j): offset of its expert + number of lower
 * tokens that selected the same expert.                                 */
int orc_buckets(int N, int E, int k, const int32_t* topk_idx, const uint8_t* placement,
                int32_t* order, int32_t* offsets, int32_t* pos);

/* O8 (SwiGLU per BASELINE north_star): one expert on one token,
 * y = Wd (silu(Wg x) * (Wu x)), fp64, no intermediate rounding.
 * wg, wu: [ffn, hidden] row-major, wd: [hidden, ffn] row-major.          */
int orc_swiglu(int hidden, int ffn, const double* x, const void* wg, const void* wu,
               const void* wd, int w_dtype, double* y);

typedef struct {
  int32_t num_experts, top_k, hidden, ffn;
  int32_t act_dtype, weight_dtype, router_dtype; /* ORC_F32 / ORC_BF16 */
  int32_t norm_topk;      /* DESIGN R-2 */
  int32_t shared_expert;  /* DESIGN R-16: one always-resident shared expert */
} orc_layer;

/* O9: out[n] = sum_j g[n,j] * FFN_{topk[n,j]}(x_n) (+ shared
 * FFN_s(x_n) with weight 1), fp64, summed over j in rank order.
 * wg/wu/wd are arrays of E per-expert pointers.  token_mask (nullable)
 * restricts the FFN/combine to tokens with mask != 0 (others get 0).    */
int orc_combine(const orc_layer* L, int N, const void* x, const int32_t* topk_idx,
                const double* gates, const void* const* wg, const void* const* wu,
                const void* const* wd, const void* swg, const void* swu, const void* swd,
                const uint8_t* token_mask, double* out);

/* Whole layer-step = O1..O9 composed in the paper's order (router ->
 * hits -> refresh/placement -> buckets -> experts -> combine).          */
int orc_moe_step(const orc_layer* L, int N, const void* x, const void* wr,
                 const void* const* wg, const void* const* wu, const void* const* wd,
                 const void* swg, const void* swu, const void* swd,
                 const uint8_t* placement_in, int step, int interval, int capacity,
                 const uint8_t* token_mask,
                 double* logits, int32_t* topk_idx, double* gates, int32_t* hits,
                 uint8_t* placement_out, int32_t* order, int32_t* offsets, int32_t* pos,
                 double* out);

/* O10 (DESIGN R-12/R-13): the expert-slot I/O model.
 * loaded[E] (in/out) marks experts whose weights sit in an HBM slot.
 * Returns counts of promotions/evictions (set differences of placements),
 * streamed experts (hit this step but not loaded) and H2D expert copies. */
typedef struct {
  int32_t promotions, evictions, experts_streamed, copies, resident_pairs, nonresident_pairs;
} orc_io;
int orc_io_step(int E, int lazy, const int32_t* hits, const uint8_t* placement_in,
                const uint8_t* placement_out, uint8_t* loaded, orc_io* io);

/* O11 (P:460-462 future work; DESIGN R-18): expert-parallel emulation over
 * P ranks in one process.  Rank r owns experts [r*E/P, (r+1)*E/P); hits are
 * global; rank r's placement = top-C_r of its own experts by global hits;
 * out = sum over ranks (in rank order) of that rank's partial combine, plus the
 * shared expert (R-16, weight 1) when L->shared_expert (swg/swu/swd, else unused). */
int orc_ep_step(const orc_layer* L, int P, int N, const void* x, const void* wr,
                const void* const* wg, const void* const* wu, const void* const* wd,
                const void* swg, const void* swu, const void* swd,
                const uint8_t* placement_in, int step, int interval, int capacity_per_rank,
                int32_t* topk_idx, int32_t* hits, uint8_t* placement_out, double* out);

/* ---------------- NEXT-1: hit-counter readings ("global hit counter"; S:242,
 * S:269-270) and the incumbent-aware tie-break.
 * mode 0 = current step (R-5); 1 = window [t_prev_refresh, t) reset at each refresh
 * (SPEC default); 2 = cumulative since block start.  In modes 1/2 step 0 of a block
 * ranks by its own hits (SPEC OracleStep0 cold start) and acc restarts.
 * orc_counter_key: the counts that rank experts at this step.
 * orc_counter_update: acc after the step (reset at refresh in mode 1, then += hits).
 * orc_placement_ex: top-C by (key desc, [incumbent first], id asc).             */
void orc_counter_key(int E, int mode, int step, const int32_t* hits, const int32_t* acc,
                     int32_t* key);
void orc_counter_update(int E, int mode, int step, int refresh, const int32_t* hits,
                        int32_t* acc);
int orc_placement_ex(int E, int capacity, const int32_t* key, int refresh, int incumbent_ties,
                     const uint8_t* placement_in, uint8_t* placement_out);

/* ---------------- NEXT-2: refresh-interval model (Eq. 4-7) ----------
 * Eq. 5: Lat_IO(tau) = c_io * (B*T/tau) * (1 - (1-d)^tau).
 * Eq. 6: Lat_miss(tau) = c_miss * T * B * f(tau), f(tau) = (1/tau) * sum_{j<tau} (1-(1-d)^j)
 *        (SPEC S:330's closed form of the paper's monotone f).  On B200 a miss streams
 *        the expert H2D (R-13), so c_miss is a per-expert H2D cost, not a CPU cost.
 * Eq. 7: tau* = argmin_{1 <= tau <= T-1} Lat_IO + Lat_miss (ties -> smallest tau). */
double orc_migration_cost(int tau, int B, int T, double d, double c_io);
double orc_miss_fraction(int tau, double d);
double orc_miss_cost(int tau, int B, int T, double d, double c_miss);
int orc_optimize_tau(int T, int B, double d, double c_io, double c_miss, double* curve);

/* ---------------- NEXT-4: routing-trace analytics -- */
/* cosine similarity of two hit-count vectors (0 if either is all-zero).            */
double orc_cosine(int E, const int32_t* a, const int32_t* b);
/* experts with hits > 0                                                            */
int orc_unique(int E, const int32_t* hits);
/* Eq. 4: d = |topB(cur) \ topB(prev)| / B, top-B by (hits desc, id asc).           */
double orc_drift(int E, int B, const int32_t* prev, const int32_t* cur);

/* NEXT-2 on B200 (DESIGN R-21): interval trade-off measured on a routing trace [T][E]. */
int orc_interval_profile(int T, int E, int B, const int32_t* counts, double* miss_lag,
                         double* mig_lag);
double orc_interval_copies_trace(int T, int tau, const double* miss_lag, const double* mig_lag);
/* NEXT-2 replay (R-24): copies of the last of `passes` back-to-back blocks of the trace. */
long orc_interval_replay(int T, int E, int B, int tau, int lazy, int passes,
                         const int32_t* counts, int32_t* copies_per_step);

#ifdef __cplusplus
}
#endif
#endif
