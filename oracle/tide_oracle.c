/*
 * tide_oracle.c -- plain, slow, obviously-correct CPU reference of one TIDE
 * MoE layer-step (arXiv 2605.20179), written from the paper.
 *
 * TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this.  It shares no code
 * with the CUDA path (paper_2605_20179_b200/csrc) and is pinned by the
 * `-m "not gpu"` tests in tests/test_oracle_pins.py against values the paper
 * and SPEC fix, closed forms, brute force and independent NumPy expressions.
 *
 * Everything is fp64, in the paper's order, one definition per function.
 * No blocking, fusion or reordering.  Citation keys: P:n = PAPER.md line n,
 * S:n = SPEC.md line n, R-x = a reading listed in DESIGN.md "Readings".
 */
#include "tide_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Threading (bench.py's cpu_baseline runs the oracle on 1 and on nproc host cores).  Only
 * loops over independent tokens are split across threads; every token's arithmetic runs in
 * the same order on one thread, so results are bit-identical for any thread count
 * (pinned by tests/test_oracle_pins.py::test_threads_bit_identical). */
void orc_set_threads(int n) {
#ifdef _OPENMP
  omp_set_num_threads(n > 0 ? n : 1);
#else
  (void)n;
#endif
}
int orc_get_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Exact conversion of a stored element to double.  bf16 is the top half of
 * an IEEE binary32, so widening is exact.                                 */
static double rd(const void* base, int dtype, size_t i) {
  if (dtype == ORC_BF16) {
    uint32_t b = (uint32_t)((const uint16_t*)base)[i] << 16;
    float f;
    memcpy(&f, &b, 4);
    return (double)f;
  }
  return (double)((const float*)base)[i];
}

/* ---------------- O1: router logits ---------------------------
 * "k experts are activated for one token" -- the router scores every expert
 * with a linear map of the token's hidden state.  Plain sum in h order.   */
int orc_router_logits(int N, int E, int hidden, const void* x, int x_dtype, const void* wr,
                      int wr_dtype, double* logits) {
  if (N < 0 || E <= 0 || hidden <= 0) return 1;
#pragma omp parallel for schedule(static)
  for (int n = 0; n < N; ++n)
    for (int e = 0; e < E; ++e) {
      double s = 0.0;
      for (int h = 0; h < hidden; ++h)
        s += rd(x, x_dtype, (size_t)n * hidden + h) * rd(wr, wr_dtype, (size_t)e * hidden + h);
      logits[(size_t)n * E + e] = s;
    }
  return 0;
}

/* expert a ranks before expert b: larger logit first, lower id on ties
 * (R-3/R-4: rank logits, not probabilities; S:88 lower id wins).          */
static int ranks_before(double la, int a, double lb, int b) {
  if (la > lb) return 1;
  if (la < lb) return 0;
  return a < b;
}

/* ---------------- O2: top-k ("E_x") -------------
 * Selection: k passes, each taking the best not-yet-taken expert.         */
int orc_topk(int N, int E, int k, const double* logits, int32_t* topk_idx) {
  if (k < 1 || k > E) return 1;
  unsigned char* taken = (unsigned char*)malloc((size_t)E);
  for (int n = 0; n < N; ++n) {
    const double* l = logits + (size_t)n * E;
    memset(taken, 0, (size_t)E);
    for (int j = 0; j < k; ++j) {
      int best = -1;
      for (int e = 0; e < E; ++e) {
        if (taken[e]) continue;
        if (best < 0 || ranks_before(l[e], e, l[best], best)) best = e;
      }
      taken[best] = 1;
      topk_idx[(size_t)n * k + j] = best;
    }
  }
  free(taken);
  return 0;
}

/* ---------------- O3: gates (BASELINE north_star "router softmax") -------
 * p = softmax(l) over all E (max-subtracted).  R-2: with norm_topk the k
 * selected probabilities are renormalised to sum to 1.                   */
int orc_gates(int N, int E, int k, const double* logits, const int32_t* topk_idx, int norm_topk,
              double* gates) {
  for (int n = 0; n < N; ++n) {
    const double* l = logits + (size_t)n * E;
    double m = l[0];
    for (int e = 1; e < E; ++e)
      if (l[e] > m) m = l[e];
    double z = 0.0;
    for (int e = 0; e < E; ++e) z += exp(l[e] - m);
    double sel = 0.0;
    for (int j = 0; j < k; ++j) sel += exp(l[topk_idx[(size_t)n * k + j]] - m) / z;
    for (int j = 0; j < k; ++j) {
      double p = exp(l[topk_idx[(size_t)n * k + j]] - m) / z;
      gates[(size_t)n * k + j] = norm_topk ? p / sel : p;
    }
  }
  return 0;
}

/* ---------------- O4: hit counter ("global hit counter") -----
 * R-5: the counter driving a refresh holds the current step's hits.       */
int orc_hits(int N, int E, int k, const int32_t* topk_idx, int32_t* hits) {
  for (int e = 0; e < E; ++e) hits[e] = 0;
  for (int n = 0; n < N; ++n)
    for (int j = 0; j < k; ++j) {
      int e = topk_idx[(size_t)n * k + j];
      if (e < 0 || e >= E) return 1;
      hits[e] += 1;
    }
  return 0;
}

/* ---------------- O5: refresh cadence (Alg. 1 line 2) ------------ */
int orc_is_refresh(int step, int interval) { return (step % interval) == 0; }

/* ---------------- O6: placement ("set to the current top-B experts",
 * P:277 "select the top experts by frequency ranking"; R-6, R-8) ---
 * rank(e) = #{e' : hits[e'] > hits[e] or (hits[e'] == hits[e] and e' < e)};
 * resident iff rank(e) < C.  Skipped steps keep the placement.    */
int orc_placement(int E, int capacity, const int32_t* hits, int refresh,
                  const uint8_t* placement_in, uint8_t* placement_out) {
  if (capacity < 1 || capacity > E) return 1;
  if (!refresh) {
    for (int e = 0; e < E; ++e) placement_out[e] = placement_in[e] ? 1 : 0;
    return 0;
  }
  for (int e = 0; e < E; ++e) {
    int rank = 0;
    for (int f = 0; f < E; ++f)
      if (hits[f] > hits[e] || (hits[f] == hits[e] && f < e)) rank++;
    placement_out[e] = rank < capacity ? 1 : 0;
  }
  return 0;
}

/* ---------------- O7: buckets (Alg. 1 lines 6-12; R-11) ------ */
int orc_buckets(int N, int E, int k, const int32_t* topk_idx, const uint8_t* placement,
                int32_t* order, int32_t* offsets, int32_t* pos) {
  int32_t* hits = (int32_t*)malloc(sizeof(int32_t) * (size_t)E);
  int32_t* first = (int32_t*)malloc(sizeof(int32_t) * (size_t)E);
  orc_hits(N, E, k, topk_idx, hits);
  int i = 0;
  for (int pass = 1; pass >= 0; --pass) /* resident first, then non-resident */
    for (int e = 0; e < E; ++e)
      if ((placement[e] ? 1 : 0) == pass) order[i++] = e;
  int32_t acc = 0;
  for (i = 0; i < E; ++i) {
    offsets[i] = acc;
    first[order[i]] = acc;
    acc += hits[order[i]];
  }
  offsets[E] = acc;
  for (int n = 0; n < N; ++n)
    for (int j = 0; j < k; ++j) {
      int e = topk_idx[(size_t)n * k + j];
      int before = 0; /* tokens n' < n that selected e (each token selects e at most once) */
      for (int m = 0; m < n; ++m)
        for (int jj = 0; jj < k; ++jj)
          if (topk_idx[(size_t)m * k + jj] == e) before++;
      pos[(size_t)n * k + j] = first[e] + before;
    }
  free(hits);
  free(first);
  return 0;
}

/* ---------------- O8: SwiGLU expert ("FFN experts"; north_star) ---
 * u = Wg x, v = Wu x, a = silu(u) * v with silu(z) = z / (1 + e^{-z}),
 * y = Wd a.  fp64 throughout (R-14: no intermediate rounding here).      */
int orc_swiglu(int hidden, int ffn, const double* x, const void* wg, const void* wu,
               const void* wd, int w_dtype, double* y) {
  double* a = (double*)malloc(sizeof(double) * (size_t)ffn);
  for (int f = 0; f < ffn; ++f) {
    double u = 0.0, v = 0.0;
    for (int h = 0; h < hidden; ++h) {
      u += rd(wg, w_dtype, (size_t)f * hidden + h) * x[h];
      v += rd(wu, w_dtype, (size_t)f * hidden + h) * x[h];
    }
    a[f] = (u / (1.0 + exp(-u))) * v;
  }
  for (int h = 0; h < hidden; ++h) {
    double s = 0.0;
    for (int f = 0; f < ffn; ++f) s += rd(wd, w_dtype, (size_t)h * ffn + f) * a[f];
    y[h] = s;
  }
  free(a);
  return 0;
}

/* ---------------- O9: combine ("re-synchronized at the end of the
 * FFN block", "output = e(x)") ------------------------------------ */
int orc_combine(const orc_layer* L, int N, const void* x, const int32_t* topk_idx,
                const double* gates, const void* const* wg, const void* const* wu,
                const void* const* wd, const void* swg, const void* swu, const void* swd,
                const uint8_t* token_mask, double* out) {
  const int H = L->hidden, F = L->ffn, k = L->top_k;
  const int per = k + (L->shared_expert ? 1 : 0); /* expert evaluations per token */
  /* y of every (token, slot) pair -- independent SwiGLUs, evaluated on any host thread --
   * then each token's sum in slot order, exactly as written in P:303. */
  double* ys = (double*)malloc(sizeof(double) * (size_t)N * per * H);
#pragma omp parallel
  {
    double* xn = (double*)malloc(sizeof(double) * (size_t)H);
#pragma omp for schedule(dynamic, 1)
    for (int q = 0; q < N * per; ++q) {
      const int n = q / per, j = q % per;
      if (token_mask && !token_mask[n]) continue;
      for (int h = 0; h < H; ++h) xn[h] = rd(x, L->act_dtype, (size_t)n * H + h);
      double* y = ys + (size_t)q * H;
      if (j < k) {
        const int e = topk_idx[(size_t)n * k + j];
        orc_swiglu(H, F, xn, wg[e], wu[e], wd[e], L->weight_dtype, y);
      } else { /* R-16: the shared expert */
        orc_swiglu(H, F, xn, swg, swu, swd, L->weight_dtype, y);
      }
    }
    free(xn);
  }
  for (int n = 0; n < N; ++n) {
    double* o = out + (size_t)n * H;
    for (int h = 0; h < H; ++h) o[h] = 0.0;
    if (token_mask && !token_mask[n]) continue;
    for (int j = 0; j < k; ++j) {
      const double g = gates[(size_t)n * k + j];
      const double* y = ys + ((size_t)n * per + j) * H;
      for (int h = 0; h < H; ++h) o[h] += g * y[h];
    }
    if (L->shared_expert) { /* R-16: weight 1, always resident, not counted */
      const double* y = ys + ((size_t)n * per + k) * H;
      for (int h = 0; h < H; ++h) o[h] += y[h];
    }
  }
  free(ys);
  return 0;
}

/* ---------------- whole layer-step, in Alg. 1's order -------------------- */
int orc_moe_step(const orc_layer* L, int N, const void* x, const void* wr,
                 const void* const* wg, const void* const* wu, const void* const* wd,
                 const void* swg, const void* swu, const void* swd,
                 const uint8_t* placement_in, int step, int interval, int capacity,
                 const uint8_t* token_mask, double* logits, int32_t* topk_idx, double* gates,
                 int32_t* hits, uint8_t* placement_out, int32_t* order, int32_t* offsets,
                 int32_t* pos, double* out) {
  const int E = L->num_experts, k = L->top_k;
  if (interval < 1 || step < 0 || k < 1 || k > E || capacity < 1 || capacity > E) return 1;
  if (orc_router_logits(N, E, L->hidden, x, L->act_dtype, wr, L->router_dtype, logits)) return 1;
  orc_topk(N, E, k, logits, topk_idx);
  orc_gates(N, E, k, logits, topk_idx, L->norm_topk, gates);
  orc_hits(N, E, k, topk_idx, hits);
  int refresh = orc_is_refresh(step, interval);
  if (!refresh) { /* S:49, S:263 budget safety on the caller's placement */
    int cnt = 0;
    for (int e = 0; e < E; ++e) cnt += placement_in[e] ? 1 : 0;
    if (cnt > capacity) return 3;
  }
  orc_placement(E, capacity, hits, refresh, placement_in, placement_out);
  orc_buckets(N, E, k, topk_idx, placement_out, order, offsets, pos);
  orc_combine(L, N, x, topk_idx, gates, wg, wu, wd, swg, swu, swd, token_mask, out);
  return 0;
}

/* ---------------- O10: I/O model (Alg. 1 lines 3-4) ----------
 * R-12: weights are read-only; eviction frees a slot (no D2H copy) and takes
 * effect after this step's compute, so an expert whose weights are in HBM at
 * the start of the step is served from HBM this step.
 * R-13: a hit expert that is not in HBM is copied host->HBM; if it is in
 * the new resident set it keeps its slot, otherwise it is streamed into
 * staging for this step only.  R-9: with lazy=0 a promoted expert is
 * copied at the refresh even without hits this step.                   */
int orc_io_step(int E, int lazy, const int32_t* hits, const uint8_t* placement_in,
                const uint8_t* placement_out, uint8_t* loaded, orc_io* io) {
  memset(io, 0, sizeof(*io));
  for (int e = 0; e < E; ++e) {
    int was = placement_in[e] ? 1 : 0, now = placement_out[e] ? 1 : 0;
    if (now && !was) io->promotions++;
    if (was && !now) io->evictions++;
    if (now) io->resident_pairs += hits[e];
    else io->nonresident_pairs += hits[e];
  }
  for (int e = 0; e < E; ++e) {
    int kept = 0;
    if (hits[e] > 0 && !loaded[e]) io->experts_streamed++;
    if (placement_out[e] && !loaded[e] && (!lazy || hits[e] > 0)) {
      io->copies++; /* copied into a slot and retained */
      kept = 1;
    } else if (!placement_out[e] && hits[e] > 0 && !loaded[e]) {
      io->copies++; /* staged for this step, not retained */
    }
    loaded[e] = (uint8_t)((loaded[e] && placement_out[e]) || kept);
  }
  return 0;
}

/* ---------------- O11: expert-parallel emulation (R-18) ------------------ */
int orc_ep_step(const orc_layer* L, int P, int N, const void* x, const void* wr,
                const void* const* wg, const void* const* wu, const void* const* wd,
                const void* swg, const void* swu, const void* swd,
                const uint8_t* placement_in, int step, int interval, int capacity_per_rank,
                int32_t* topk_idx, int32_t* hits, uint8_t* placement_out, double* out) {
  const int E = L->num_experts, k = L->top_k, H = L->hidden;
  if (P < 1 || E % P != 0) return 1;
  const int El = E / P;
  if (capacity_per_rank < 1 || capacity_per_rank > El) return 1;
  double* logits = (double*)malloc(sizeof(double) * (size_t)N * E);
  double* gates = (double*)malloc(sizeof(double) * (size_t)N * k);
  double* part = (double*)malloc(sizeof(double) * (size_t)N * H);
  double* xn = (double*)malloc(sizeof(double) * (size_t)H);
  double* y = (double*)malloc(sizeof(double) * (size_t)H);
  orc_router_logits(N, E, H, x, L->act_dtype, wr, L->router_dtype, logits);
  orc_topk(N, E, k, logits, topk_idx);
  orc_gates(N, E, k, logits, topk_idx, L->norm_topk, gates);
  orc_hits(N, E, k, topk_idx, hits);
  int refresh = orc_is_refresh(step, interval);
  for (int r = 0; r < P; ++r) /* each rank places only its own experts */
    orc_placement(El, capacity_per_rank, hits + (size_t)r * El, refresh,
                  placement_in + (size_t)r * El, placement_out + (size_t)r * El);
  for (size_t i = 0; i < (size_t)N * H; ++i) out[i] = 0.0;
  for (int r = 0; r < P; ++r) {
    for (size_t i = 0; i < (size_t)N * H; ++i) part[i] = 0.0;
#pragma omp parallel
    {
      double* xt = (double*)malloc(sizeof(double) * (size_t)H);
      double* yt = (double*)malloc(sizeof(double) * (size_t)H);
#pragma omp for schedule(dynamic, 1)
      for (int n = 0; n < N; ++n) {
        for (int h = 0; h < H; ++h) xt[h] = rd(x, L->act_dtype, (size_t)n * H + h);
        for (int j = 0; j < k; ++j) {
          int e = topk_idx[(size_t)n * k + j];
          if (e / El != r) continue;
          orc_swiglu(H, L->ffn, xt, wg[e], wu[e], wd[e], L->weight_dtype, yt);
          for (int h = 0; h < H; ++h) part[(size_t)n * H + h] += gates[(size_t)n * k + j] * yt[h];
        }
      }
      free(xt);
      free(yt);
    }
    for (size_t i = 0; i < (size_t)N * H; ++i) out[i] += part[i];
  }
  if (L->shared_expert) { /* R-16: the token's own rank adds its shared expert, weight 1 */
    for (int n = 0; n < N; ++n) {
      for (int h = 0; h < H; ++h) xn[h] = rd(x, L->act_dtype, (size_t)n * H + h);
      orc_swiglu(H, L->ffn, xn, swg, swu, swd, L->weight_dtype, y);
      for (int h = 0; h < H; ++h) out[(size_t)n * H + h] += y[h];
    }
  }
  free(logits);
  free(gates);
  free(part);
  free(xn);
  free(y);
  return 0;
}

/* ---------------- NEXT-2: Eq. 5 --------------------------------------- */
double orc_migration_cost(int tau, int B, int T, double d, double c_io) {
  return c_io * ((double)B * (double)T / (double)tau) * (1.0 - pow(1.0 - d, (double)tau));
}

/* f(tau): mean fraction of the placement made stale by drift over an interval,
 * (1/tau) sum_{j=0}^{tau-1} (1 - (1-d)^j)  (Eq. 6 is stated only as monotone). */
double orc_miss_fraction(int tau, double d) {
  double s = 0.0;
  for (int j = 0; j < tau; ++j) s += 1.0 - pow(1.0 - d, (double)j);
  return s / (double)tau;
}

/* Eq. 6 with the miss cost of this build (R-13). */
double orc_miss_cost(int tau, int B, int T, double d, double c_miss) {
  return c_miss * (double)T * (double)B * orc_miss_fraction(tau, d);
}

/* Eq. 7: exhaustive scan of tau in [1, T-1] ("greedy search");
 * curve[tau-1] = total cost; ties -> smallest tau. */
int orc_optimize_tau(int T, int B, double d, double c_io, double c_miss, double* curve) {
  int best = 1;
  double best_c = 0.0;
  for (int tau = 1; tau <= (T > 1 ? T - 1 : 1); ++tau) {
    double c = orc_migration_cost(tau, B, T, d, c_io) + orc_miss_cost(tau, B, T, d, c_miss);
    if (curve) curve[tau - 1] = c;
    if (tau == 1 || c < best_c) {
      best = tau;
      best_c = c;
    }
  }
  return best;
}

/* ---------------- NEXT-4: cosine similarity of count vectors ----------- */
double orc_cosine(int E, const int32_t* a, const int32_t* b) {
  double ab = 0.0, aa = 0.0, bb = 0.0;
  for (int e = 0; e < E; ++e) {
    ab += (double)a[e] * (double)b[e];
    aa += (double)a[e] * (double)a[e];
    bb += (double)b[e] * (double)b[e];
  }
  if (aa == 0.0 || bb == 0.0) return 0.0;
  return ab / (sqrt(aa) * sqrt(bb));
}

int orc_unique(int E, const int32_t* hits) {
  int u = 0;
  for (int e = 0; e < E; ++e) u += hits[e] > 0;
  return u;
}

/* Eq. 4: drift of the optimal (top-B) placement between two steps. */
double orc_drift(int E, int B, const int32_t* prev, const int32_t* cur) {
  uint8_t* a = (uint8_t*)malloc((size_t)E);
  uint8_t* b = (uint8_t*)malloc((size_t)E);
  orc_placement(E, B, prev, 1, a, a);
  orc_placement(E, B, cur, 1, b, b);
  int diff = 0;
  for (int e = 0; e < E; ++e) diff += (b[e] && !a[e]);
  free(a);
  free(b);
  return (double)diff / (double)B;
}

/* ---------------- NEXT-1: counters ("counts accumulated over [t_prev_refresh, t)",
 * reset at refresh; S:269 cumulative variant; S:270 current-step "oracle mode" = R-5) -- */
void orc_counter_key(int E, int mode, int step, const int32_t* hits, const int32_t* acc,
                     int32_t* key) {
  for (int e = 0; e < E; ++e) key[e] = (mode == 0 || step == 0) ? hits[e] : acc[e];
}

void orc_counter_update(int E, int mode, int step, int refresh, const int32_t* hits,
                        int32_t* acc) {
  if (mode == 0) return;
  for (int e = 0; e < E; ++e) {
    if (step == 0 || (mode == 1 && refresh)) acc[e] = 0;
    acc[e] += hits[e];
  }
}

/* Top-C with the incumbent-aware tie-break: among equal keys, experts
 * already in the input placement rank first, then lower id. */
int orc_placement_ex(int E, int capacity, const int32_t* key, int refresh, int incumbent_ties,
                     const uint8_t* placement_in, uint8_t* placement_out) {
  if (capacity < 1 || capacity > E) return 1;
  if (!refresh) {
    for (int e = 0; e < E; ++e) placement_out[e] = placement_in[e] ? 1 : 0;
    return 0;
  }
  for (int e = 0; e < E; ++e) {
    int rank = 0;
    for (int f = 0; f < E; ++f) {
      int before;
      if (key[f] != key[e]) {
        before = key[f] > key[e];
      } else if (incumbent_ties && ((placement_in[f] != 0) != (placement_in[e] != 0))) {
        before = placement_in[f] != 0;
      } else {
        before = f < e;
      }
      rank += before;
    }
    placement_out[e] = rank < capacity ? 1 : 0;
  }
  return 0;
}

/* ---------------- NEXT-2 on B200 (DESIGN R-21): the interval trade-off on a routing trace --
 * miss_lag[j] = mean over t of |{e : counts[t+j][e] > 0} \ topB(counts[t])| (hit experts
 * outside a placement refreshed j steps earlier, streamed per R-13), mig_lag[j] = mean over t
 * of |topB(counts[t+j]) \ topB(counts[t])| (promotions at a refresh of a j-step-old
 * placement: Eq. 4's drift at lag j, times B), t = 0..T-1-j; topB is O6's rule.          */
int orc_interval_profile(int T, int E, int B, const int32_t* counts, double* miss_lag,
                         double* mig_lag) {
  if (T < 1 || E < 1 || B < 1 || B > E) return 1;
  uint8_t* top = (uint8_t*)malloc((size_t)T * E);
  for (int t = 0; t < T; ++t)
    orc_placement(E, B, counts + (size_t)t * E, 1, top + (size_t)t * E, top + (size_t)t * E);
  for (int j = 0; j < T; ++j) {
    long miss = 0, mig = 0;
    for (int t = 0; t + j < T; ++t)
      for (int e = 0; e < E; ++e) {
        if (counts[(size_t)(t + j) * E + e] > 0 && !top[(size_t)t * E + e]) miss++;
        if (top[(size_t)(t + j) * E + e] && !top[(size_t)t * E + e]) mig++;
      }
    miss_lag[j] = (double)miss / (double)(T - j);
    mig_lag[j] = (double)mig / (double)(T - j);
  }
  free(top);
  return 0;
}

/* Copies over a block of T steps refreshing every tau steps: T/tau intervals, each one
 * refresh (mig_lag[tau] promotions) and tau steps of misses (miss_lag[0..tau-1]).        */
double orc_interval_copies_trace(int T, int tau, const double* miss_lag, const double* mig_lag) {
  double per = mig_lag[tau];
  for (int j = 0; j < tau; ++j) per += miss_lag[j];
  return (double)T / (double)tau * per;
}

/* ---------------- NEXT-2 replay (DESIGN R-24): the copies an interval causes on a trace ----
 * Alg. 1 lines 3-4 run step by step over a recorded routing trace: at every
 * step t of a block, refresh iff t % tau == 0 (O3), placement by O6 (R-5 current-step
 * counts, R-8 ties), expert copies by O10 (R-9 eager/lazy, R-12 eviction after the step,
 * R-13 streaming).  `passes` blocks of the same trace run back to back, the placement and
 * the loaded set carried from block to block, nothing loaded before the first block;
 * the copies of the LAST pass are returned (per step in copies_per_step, may be NULL).   */
long orc_interval_replay(int T, int E, int B, int tau, int lazy, int passes,
                         const int32_t* counts, int32_t* copies_per_step) {
  if (T < 1 || E < 1 || B < 1 || B > E || tau < 1 || passes < 1) return -1;
  uint8_t* pl = (uint8_t*)calloc((size_t)E, 1);
  uint8_t* npl = (uint8_t*)calloc((size_t)E, 1);
  uint8_t* loaded = (uint8_t*)calloc((size_t)E, 1);
  long total = 0;
  for (int pass = 0; pass < passes; ++pass)
    for (int t = 0; t < T; ++t) {
      const int32_t* hits = counts + (size_t)t * E;
      orc_placement(E, B, hits, orc_is_refresh(t, tau), pl, npl);
      orc_io io;
      orc_io_step(E, lazy, hits, pl, npl, loaded, &io);
      memcpy(pl, npl, (size_t)E);
      if (pass == passes - 1) {
        total += io.copies;
        if (copies_per_step) copies_per_step[t] = io.copies;
      }
    }
  free(pl);
  free(npl);
  free(loaded);
  return total;
}
