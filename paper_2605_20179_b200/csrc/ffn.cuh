// ffn.cuh -- a7/a8/a9: grouped SwiGLU expert FFN on tcgen05 tensor cores fed by TMA.
//
//   phase 1 (per work entry w, F-tile t):  u = Wg[t] X_w^T, v = Wu[t] X_w^T   (TMEM, fp32)
//                                          h[w, t] = bf16(silu(u) * v)         (R-14)
//   phase 2 (per entry w, H-tile t):       y[w, t] = Wd[t] h_w^T                (TMEM -> fp32 y)
//
// The expert weights are the MMA M operand (128 rows per tile, streamed once per
// work entry, L2 evict-first); the entry's tokens are the N operand (m <= 128
// rows, padded to a multiple of 16, L2 evict-last).  Because m is small the
// kernel is a weight stream: it is judged by HBM GB/s.
//
// Persistent, warp-specialised, one CTA per SM (192 threads):
//   warp 0 lane 0 : scheduler + TMA producer (global atomic work counter; items are
//                   all phase-1 items in entry order, then all phase-2 items)
//   warp 1 lane 0 : tcgen05.mma issuer (single thread), commits to mbarriers
//   warps 2..5    : epilogue (TMEM -> registers -> global); warp 2 owns TMEM alloc
// A phase-2 item waits (acquire) on its entry's phase-1 counter; phase-1 items are
// all claimed before any phase-2 item, so the wait cannot deadlock.
#pragma once
#include <type_traits>

#include "ptx.cuh"
#include "route.cuh"

namespace tide {

constexpr int kFfnThreads = 192;
constexpr int kStages = 4;
constexpr int kItemSlots = 4;
constexpr int kTileM = 128;
constexpr int kATile = kTileM * 128;           // 16 KB: 128 rows x 128 B (one K block)
constexpr int kBTile = kMaxTok * 128;          // 16 KB: up to 128 token rows x 128 B
constexpr int kStageBytes = 2 * kATile + kBTile;
constexpr int kMaxEntriesSmem = 1280;          // work entries per CTA at most (E + N*k/128 + ...);
                                               // a launch allocates its context's max_entries
constexpr int kFfnSmemBytes = kStages * kStageBytes + 2048 + 4 * kMaxTok + 16 * kMaxEntriesSmem;

struct FfnParams {
  CUtensorMap map_gu;    // routed pool viewed as rows of H elements (gate/up rows)
  CUtensorMap map_d;     // routed pool viewed as rows of F elements (down rows)
  CUtensorMap map_gu_s;  // shared expert, rows of H
  CUtensorMap map_d_s;   // shared expert, rows of F
  CUtensorMap map_x;     // x_in [maxN, H], box = 1 row (tile::gather4)
  CUtensorMap map_h;     // h_perm [rows, F]
  // work entries {weight slot, first h/y row, m | flags << 16, token-list index};
  // flags bit0: shared-expert weights, bit1: identity token list (token = index + j).
  // build mode (cnt != nullptr): every CTA builds the list from the per-expert counts:
  // experts in id order with m > 0 and (slot_of == nullptr or slot_of[e] >= 0), rows
  // off[e] = prefix of counts in id order, then the shared expert (rows N*k + n).
  const int* cnt;        // [E] per-expert token counts (build mode), or [2][E] with par
  const int* par;        // nullable: route's parity word, this step's counts = cnt[par^1]
  L2Prefetch pf;         // NEXT-3: issued by each CTA once it has no more work (route.cuh)
  L2Prefetch pf_self;    // NEXT-3: this layer's likely experts past the previous layer's range,
                         // issued before the wait on the routing (HBM is idle until then)
  const int* slot_of;    // [E] pool slot (nullptr: slot = e)
  int* off_out;          // [E] row offsets written by CTA 0 (build mode; read by combine)
  const int4* entries;   // global mode: host-built list
  const int* n_entries;
  const int* list;       // [E * maxN] token lists
  int* sched;
  int* done;
  void* h_out;
  float* y_out;
  int H, F, E, maxN, N, k, shared;
  unsigned long long* trace;  // debug: per CTA [entry, work list ready, producer done, epilogue done, items]
  unsigned long long* itrace;  // debug: per CTA, 64 items x {claim, kind<<32|entry, dep met, issued}
  // Peer-memory EP (tide_ffn_kernel<T, true>): the phase-2 epilogue stores each routed pair's
  // y row straight into the owning rank's ypair[n*k + j] over peer memory -- the combine's
  // exchange fused into the GEMM epilogue; every CTA then delivers a slice of the local
  // experts' counts into every rank's hits_all and arrives once on each rank's combine
  // counter after its own release.  Shared-expert rows stay local (y_out).
  int ep_P, ep_e0, ep_El;
  const unsigned* ep_dst; // [El][rows_all] per list slot: owner rank << 28 | pair row n*k + j
  const int* ep_cnt_l;    // [2][El] local experts' counts by parity (global hits of those
                          // experts); this step's half is [par ^ 1] once the route flipped par
  const int* ep_par;      // step parity word (flipped by the route kernel)
  char* ep_base[8];       // symmetric regions of every rank
  size_t ep_off_ypair, ep_off_hits, ep_off_ctr;
  int shared_row0;       // first h/y row of the shared expert's tokens (N*k single-device)
  int shared_tok0;       // token id of its first row (0 single-device, rank*maxN under EP)
};

struct FfnItem {
  int kind;  // 0 gate/up, 1 down, -1 end
  int tile, slot, off, m, flags, entry, tokbase;
};

template <typename T, bool EP>
__global__ void __launch_bounds__(kFfnThreads, 1)
    tide_ffn_kernel(const __grid_constant__ FfnParams p) {
  constexpr bool kTF32 = std::is_same<T, float>::value;
  constexpr int EB = sizeof(T);
  constexpr int BK = 128 / EB;  // elements per K block (one 128-byte swizzle row)
  constexpr int UK = 32 / EB;   // elements per MMA K step
  constexpr int KSTEPS = BK / UK;

  extern __shared__ uint8_t ffn_smem_raw[];
  // 1024-byte aligned (SW128 tiles); offsetting the shared array itself keeps the shared
  // state space visible to the compiler (LDS/STS, not generic loads/stores)
  uint8_t* smem = ffn_smem_raw + ((1024u - (smem_u32(ffn_smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* ifull = tempty + 2;
  uint64_t* iempty = ifull + kItemSlots;
  FfnItem* items = reinterpret_cast<FfnItem*>(iempty + kItemSlots);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(items + kItemSlots);
  int* s_tok = reinterpret_cast<int*>(tmem_slot + 4);  // producer: row ids of the current item
  int4* s_ent = reinterpret_cast<int4*>(s_tok + kMaxTok);  // build mode: this CTA's work list

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long* tr = p.trace ? p.trace + 8 * blockIdx.x : nullptr;
  if (tr && threadIdx.x == 0) tr[0] = globaltimer_ns();
  const int H = p.H, F = p.F;
  const int FT = (F + kTileM - 1) / kTileM, HT = (H + kTileM - 1) / kTileM;
  const int KB1 = H / BK, KB2 = F / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 4); }
    for (int i = 0; i < kItemSlots; ++i) { mbar_init(&ifull[i], 1); mbar_init(&iempty[i], 5); }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&p.map_gu);
    tma_prefetch_desc(&p.map_d);
    tma_prefetch_desc(&p.map_x);
    tma_prefetch_desc(&p.map_h);
  }
  if (warp == 2) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // routing (counts, token lists, x_in) comes from the preceding grid; the dependent grid
  // (combine) may launch once every CTA is past that wait, so it can read the routing it
  // needs (top-k, slots, gates) before its own wait on this grid
  // the MMA warp is idle until the first item: while the routing is still being computed it
  // pulls this CTA's share of this layer's likely experts (beyond what the previous layer's
  // FFN tail prefetched) into L2
  if (warp == 1) issue_l2_prefetch(p.pf_self, blockIdx.x + (long long)gridDim.x * lane, (long long)gridDim.x * 32);
  if (warp == 0) pdl_wait();
  __syncthreads();
  pdl_trigger();
  if (tr && threadIdx.x == 0) tr[5] = globaltimer_ns();

  // Work list (build mode): every thread of the CTA takes a contiguous range of experts, loads
  // their counts in one batch (both count halves, the parity word and the slots: one L2 round
  // trip, no dependent chain), then a CTA-wide exclusive scan of (rows, entries) places each
  // expert's entries in s_ent and (CTA 0) its first FFN row in off_out.
  __shared__ int s_wsum[2][kFfnThreads / 32];
  __shared__ int s_nent;
  if (p.cnt) {
    const int E = p.E, t = threadIdx.x;
    constexpr int PER = 4;  // experts per thread in the batched path (E <= 4 * 192)
    const int per = (E + kFfnThreads - 1) / kFfnThreads;
    int rows = 0, nent = 0;
    int m4[PER], s4[PER];
    const int e0 = min(E, t * per), e1 = min(E, e0 + per);
    if (per <= PER) {
      int mb[PER];
      const int pr = p.par ? __ldcg(p.par) : 1;
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int e = e0 + i;
        const bool ok = e < e1;
        m4[i] = ok ? __ldcg(p.cnt + e) : 0;
        mb[i] = (ok && p.par) ? __ldcg(p.cnt + E + e) : 0;
        s4[i] = ok ? (p.slot_of ? __ldcg(p.slot_of + e) : e) : -1;
      }
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        if (pr == 0) m4[i] = mb[i];  // this step's counts live in cnt[par ^ 1]
        rows += m4[i];
        nent += (m4[i] > 0 && s4[i] >= 0) ? (m4[i] + kMaxTok - 1) / kMaxTok : 0;
      }
    } else {  // very large E: per-expert loop (not on the benchmarked shapes)
      const int* cnt = p.par ? p.cnt + (__ldcg(p.par) ^ 1) * E : p.cnt;
      for (int e = e0; e < e1; ++e) {
        const int m = __ldcg(cnt + e);
        const bool in_hbm = !p.slot_of || __ldcg(p.slot_of + e) >= 0;
        rows += m;
        nent += (m > 0 && in_hbm) ? (m + kMaxTok - 1) / kMaxTok : 0;
      }
    }
    int rows_x = rows, ent_x = nent;  // warp inclusive scans, then the warps' prefixes
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, rows_x, o), b = __shfl_up_sync(0xffffffffu, ent_x, o);
      if (lane >= o) { rows_x += a; ent_x += b; }
    }
    if (lane == 31) { s_wsum[0][warp] = rows_x; s_wsum[1][warp] = ent_x; }
    __syncthreads();
    // the shared expert's entries go first (its items do not depend on the routing, and its
    // y slices are then not the last ones of a token), the routed entries after them
    const int n_sh = p.shared ? (p.N + kMaxTok - 1) / kMaxTok : 0;
    int row = rows_x - rows, ei = n_sh + ent_x - nent;
    for (int w = 0; w < warp; ++w) { row += s_wsum[0][w]; ei += s_wsum[1][w]; }
    if (per <= PER) {
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int e = e0 + i, m = m4[i];
        if (e < e1) {
          if (blockIdx.x == 0) p.off_out[e] = row;
          if (m > 0 && s4[i] >= 0)
            for (int c = 0; c * kMaxTok < m; ++c)
              s_ent[ei++] = make_int4(s4[i], row + c * kMaxTok, min(kMaxTok, m - c * kMaxTok),
                                      e * p.maxN + c * kMaxTok);
          row += m;
        }
      }
    } else {
      const int* cnt = p.par ? p.cnt + (__ldcg(p.par) ^ 1) * E : p.cnt;
      for (int e = e0; e < e1; ++e) {
        const int m = __ldcg(cnt + e);
        const int slot = p.slot_of ? __ldcg(p.slot_of + e) : e;
        if (blockIdx.x == 0) p.off_out[e] = row;
        if (m > 0 && slot >= 0)
          for (int c = 0; c * kMaxTok < m; ++c)
            s_ent[ei++] = make_int4(slot, row + c * kMaxTok, min(kMaxTok, m - c * kMaxTok),
                                    e * p.maxN + c * kMaxTok);
        row += m;
      }
    }
    int n_r = 0;  // routed entries in total
    for (int w = 0; w < kFfnThreads / 32; ++w) n_r += s_wsum[1][w];
    for (int c = t; c < n_sh; c += kFfnThreads)
      s_ent[c] = make_int4(0, p.shared_row0 + c * kMaxTok,
                                 min(kMaxTok, p.N - c * kMaxTok) | (3 << 16),
                                 p.shared_tok0 + c * kMaxTok);
    if (t == 0) s_nent = n_r + n_sh;
    __syncthreads();
  }

  if (warp == 0) {
    // ===================== scheduler + TMA producer =====================
    int n_ent;
    const int4* ents = p.entries;
    if (p.cnt) {
      n_ent = s_nent;
      ents = s_ent;
    } else {
      n_ent = *p.n_entries;
    }
    // warp-wide producer: lane 0 schedules, waits and loads the weight tiles; lane i
    // issues the i-th token-row load of each stage (gather4 / box), so large entries are
    // not bound by a single thread's TMA issue rate
    if (tr && lane == 0) tr[1] = globaltimer_ns();
    int n_items = 0;
    const int n1 = n_ent * FT, total = n1 + n_ent * HT;
    const uint64_t pol_w = policy_evict_first(), pol_a = policy_evict_last();
    int stage = 0, islot = 0;
    uint32_t sphase = 0, iphase = 0;
    // item i of the first wave is CTA i's (no counter round trip before the first loads);
    // every later item comes from the shared counter, offset past the first wave
    int it = blockIdx.x;
    // phase-2 dependencies: entries [ready_base, ready_base + 32) whose phase-1 counters this
    // warp has acquired complete (bit i = entry ready_base + i) need no round trip
    unsigned ready = 0u;
    int ready_base = 0;
    while (true) {
      unsigned long long* itr = (p.itrace && n_items < 64)
                                    ? p.itrace + 4 * (64 * (size_t)blockIdx.x + n_items) : nullptr;
      if (itr && lane == 0) itr[0] = globaltimer_ns();
      FfnItem item;
      item.kind = -1;
      if (it < total) {
        int entry, tile;
        if (it < n1) { item.kind = 0; entry = it / FT; tile = it % FT; }
        else { item.kind = 1; entry = (it - n1) / HT; tile = (it - n1) % HT; }
        const int4 en = ents[entry];
        item.tile = tile; item.slot = en.x; item.off = en.y; item.m = en.z & 0xFFFF;
        item.flags = en.z >> 16; item.tokbase = en.w;
        item.entry = entry;
      }
      if (lane == 0) {
        mbar_wait(&iempty[islot], iphase ^ 1);
        items[islot] = item;
        mbar_arrive(&ifull[islot]);
      }
      __syncwarp();
      if (++islot == kItemSlots) { islot = 0; iphase ^= 1; }
      if (item.kind < 0) break;
      ++n_items;
      if (itr && lane == 0) itr[1] = ((unsigned long long)item.kind << 32) | (unsigned)item.entry;
      const int nbox = (item.m + 15) >> 4;
      if (item.kind == 0) {
        if (itr && lane == 0) itr[2] = globaltimer_ns();
        // token rows of this entry, gathered straight from x_in: lane i loads rows
        // 4i..4i+3 (rows past m repeat the last token; their MMA columns are discarded)
        const int ng = (item.m + 3) >> 2;
        int4 rows4 = make_int4(0, 0, 0, 0);
        if (lane < ng) {
          int rr[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int jj = item.tokbase + min(4 * lane + i, item.m - 1);
            rr[i] = (item.flags & 2) ? jj : __ldcg(p.list + jj);
          }
          rows4 = make_int4(rr[0], rr[1], rr[2], rr[3]);
        }
        const CUtensorMap* ma = (item.flags & 1) ? &p.map_gu_s : &p.map_gu;
        const int rowg = item.slot * 3 * F + item.tile * kTileM;
        const int rowu = rowg + F;
        for (int kb = 0; kb < KB1; ++kb) {
          uint8_t* sa = smem + stage * kStageBytes;
          uint8_t* sb = sa + 2 * kATile;
          if (lane == 0) {
            mbar_wait(&empty[stage], sphase ^ 1);
            mbar_arrive_expect_tx(&full[stage], 2 * kATile + ng * 512);
            tma_load_2d(sa, ma, &full[stage], kb * BK, rowg, pol_w);
            tma_load_2d(sa + kATile, ma, &full[stage], kb * BK, rowu, pol_w);
          }
          __syncwarp();
          if (lane < ng) tma_gather4(sb + lane * 512, &p.map_x, &full[stage], kb * BK, rows4, pol_a);
          if (++stage == kStages) { stage = 0; sphase ^= 1; }
        }
      } else {
        // h of this entry must be complete (all FT phase-1 tiles, possibly on other SMs)
        // The warp acquires the counters of 32 entries at once (lane i: entry item.entry + i):
        // later items of entries already seen complete skip the round trip (phase-2 items are
        // claimed in entry order, so the next few items of this CTA usually fall in the window;
        // +1.0% on the headline).  Complete once, complete for the launch.
        const int rel = item.entry - ready_base;
        if (rel < 0 || rel >= 32 || !((ready >> rel) & 1u)) {  // warp-uniform
          ready_base = item.entry;
          const int e = item.entry + lane;
          uint64_t t0 = 0;
          while (true) {
            ready = __ballot_sync(0xffffffffu, e < n_ent && ld_acquire_gpu(p.done + e) >= FT);
            if (ready & 1u) break;
            if (t0 == 0) t0 = globaltimer_ns();
            __nanosleep(64);
            if (lane == 0 && globaltimer_ns() - t0 > 4000000000ull) {
              printf("tide: ffn dependency watchdog entry %d\n", item.entry);
              __trap();
            }
          }
        }
        __syncwarp();  // the acquiring lanes' barrier orders every lane's loads below after it
        if (itr && lane == 0) itr[2] = globaltimer_ns();
        fence_proxy_async_global();  // generic-proxy h stores of other CTAs -> TMA reads
        const CUtensorMap* ma = (item.flags & 1) ? &p.map_d_s : &p.map_d;
        const int rowd = item.slot * 3 * H + 2 * H + item.tile * kTileM;
        const bool dual = item.m <= 64;
        for (int kb = 0; kb < KB2; kb += dual ? 2 : 1) {
          const int nk = (dual && kb + 1 < KB2) ? 2 : 1;
          uint8_t* sa = smem + stage * kStageBytes;
          uint8_t* sb = sa + 2 * kATile;
          if (lane == 0) {
            mbar_wait(&empty[stage], sphase ^ 1);
            mbar_arrive_expect_tx(&full[stage], nk * (kATile + nbox * 2048));
            for (int q = 0; q < nk; ++q)
              tma_load_2d(sa + q * kATile, ma, &full[stage], (kb + q) * BK, rowd, pol_w);
          }
          __syncwarp();
          if (lane < nk * nbox) {
            const int q = lane / nbox, b = lane % nbox;
            tma_load_2d(sb + (q * nbox + b) * 2048, &p.map_h, &full[stage], (kb + q) * BK,
                        item.off + 16 * b, pol_a);
          }
          if (++stage == kStages) { stage = 0; sphase ^= 1; }
        }
      }
      if (itr && lane == 0) itr[3] = globaltimer_ns();
      {  // the next item: a claim on the shared counter (claiming earlier, one item ahead or at
         // the item's last stage, was measured slower: DESIGN.md section 11)
        int raw = 0;
        if (lane == 0) raw = atomicAdd(p.sched, 1);
        it = __shfl_sync(0xffffffffu, (int)gridDim.x + raw, 0);
      }
    }
    if (tr && lane == 0) { tr[2] = globaltimer_ns(); tr[4] = n_items; }
    // NEXT-3 cross-layer prefetch: this CTA has no more work, so its share of the next
    // layer's likely experts (that layer's hit experts at its previous step, in the order its
    // FFN claims them: the shared expert, then ascending id) is pulled into L2 while the FFN
    // drains and the combine / next routing leave HBM idle.  Piece i of the byte range goes
    // to CTA i % grid, so the first CTAs to finish cover the first-claimed experts first.
    // A cache hint only: values are unaffected.
    issue_l2_prefetch(p.pf, blockIdx.x + (long long)gridDim.x * lane, (long long)gridDim.x * 32);
  } else if (warp == 1 && lane == 0) {
    // ===================== MMA issuer (one thread) =====================
    int stage = 0, islot = 0, acc = 0;
    uint32_t sphase = 0, iphase = 0, aphase = 0;
    while (true) {
      mbar_wait(&ifull[islot], iphase);
      const FfnItem item = items[islot];
      mbar_arrive(&iempty[islot]);
      if (++islot == kItemSlots) { islot = 0; iphase ^= 1; }
      if (item.kind < 0) break;
      mbar_wait(&tempty[acc], aphase ^ 1);
      tc_fence_after();
      const int nbox = (item.m + 15) >> 4;
      const uint32_t idesc = idesc_m128((uint32_t)nbox * 16u, kTF32);
      const uint32_t dcol = tmem + (uint32_t)acc * 256u;
      if (item.kind == 0) {
        for (int kb = 0; kb < KB1; ++kb) {
          mbar_wait(&full[stage], sphase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * kStageBytes);
          const uint64_t dg = smem_desc_sw128(sa), du = smem_desc_sw128(sa + kATile);
          const uint64_t db = smem_desc_sw128(sa + 2 * kATile);
#pragma unroll
          for (int k = 0; k < KSTEPS; ++k) {
            const uint32_t accum = (kb | k) != 0;
            tc_mma<kTF32>(dcol, dg + 2 * k, db + 2 * k, idesc, accum);
            tc_mma<kTF32>(dcol + 128, du + 2 * k, db + 2 * k, idesc, accum);
          }
          tc_commit(&empty[stage]);
          if (++stage == kStages) { stage = 0; sphase ^= 1; }
        }
      } else {
        const bool dual = item.m <= 64;
        for (int kb = 0; kb < KB2; kb += dual ? 2 : 1) {
          const int nk = (dual && kb + 1 < KB2) ? 2 : 1;
          mbar_wait(&full[stage], sphase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * kStageBytes);
          for (int q = 0; q < nk; ++q) {
            const uint64_t da = smem_desc_sw128(sa + q * kATile);
            const uint64_t db = smem_desc_sw128(sa + 2 * kATile + q * nbox * 2048);
#pragma unroll
            for (int k = 0; k < KSTEPS; ++k)
              tc_mma<kTF32>(dcol, da + 2 * k, db + 2 * k, idesc, ((kb + q) | k) != 0);
          }
          tc_commit(&empty[stage]);
          if (++stage == kStages) { stage = 0; sphase ^= 1; }
        }
      }
      tc_commit(&tfull[acc]);
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
    }
  } else if (warp >= 2) {
    // ===================== epilogue (4 warps, one TMEM lane quarter each) =====================
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    int islot = 0, acc = 0;
    uint32_t iphase = 0, aphase = 0;
    while (true) {
      mbar_wait(&ifull[islot], iphase);
      const FfnItem item = items[islot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&iempty[islot]);
      if (++islot == kItemSlots) { islot = 0; iphase ^= 1; }
      if (item.kind < 0) break;
      // EP: the first 16 rows' destinations are fetched while the MMAs still run
      unsigned d0[16];
      if (EP && item.kind == 1 && !(item.flags & 2)) {
#pragma unroll
        for (int i = 0; i < 16; ++i)  // same address in every thread: broadcast loads
          d0[i] = i < item.m ? __ldg(p.ep_dst + item.tokbase + i) : 0u;
      }
      mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
      const uint32_t tbase = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)acc * 256u;
      if (item.kind == 0) {
        const int f = item.tile * kTileM + row;
        T* hcol = reinterpret_cast<T*>(p.h_out) + f;
        for (int c0 = 0; c0 < item.m; c0 += 16) {
          float g[16], u[16];
          tmem_ld16(tbase + c0, g);
          tmem_ld16(tbase + 128 + c0, u);
          if (f < F) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              if (c0 + i < item.m) {
                const float s = g[i] / (1.0f + __expf(-g[i]));
                hcol[(size_t)(item.off + c0 + i) * F] = from_f32<T>(s * u[i]);
              }
            }
          }
        }
      } else if (EP && !(item.flags & 2)) {  // EP: y of pair (n, j) -> owner's ypair[n*k + j]
        const int h = item.tile * kTileM + row;
        for (int c0 = 0; c0 < item.m; c0 += 16) {
          float v[16];
          unsigned d[16];
#pragma unroll
          for (int i = 0; i < 16; ++i)  // same address in every thread: broadcast loads
            d[i] = c0 == 0 ? d0[i] : (c0 + i < item.m ? __ldg(p.ep_dst + item.tokbase + c0 + i) : 0u);
          tmem_ld16(tbase + c0, v);
          if (h < H) {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (c0 + i < item.m)
                reinterpret_cast<float*>(p.ep_base[d[i] >> 28] + p.ep_off_ypair)
                    [(size_t)(d[i] & 0x0FFFFFFFu) * H + h] = v[i];
          }
        }
      } else {
        const int h = item.tile * kTileM + row;
        float* ycol = p.y_out + h;
        for (int c0 = 0; c0 < item.m; c0 += 16) {
          float v[16];
          tmem_ld16(tbase + c0, v);
          if (h < H) {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (c0 + i < item.m) ycol[(size_t)(item.off + c0 + i) * H] = v[i];
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
      if (item.kind == 0) {  // publish this F-tile of h to phase-2 consumers on any SM
        named_bar_sync(1, 128);  // the 128 epilogue threads' h stores, then one release
        if (warp == 2 && lane == 0) red_release_gpu_add(p.done + item.entry, 1);
      }
    }
  }
  if (tr && threadIdx.x == 64) tr[3] = globaltimer_ns();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
  if constexpr (EP) {
    // every CTA (no last-CTA tail): its slice of the local experts' counts into every rank's
    // hits_all, then one release (system scope when a peer is another GPU) covering the CTA's
    // peer y stores (ordered before it by the barrier above) and one arrival on every rank's
    // combine counter; the final kernel waits for the sum of the ranks' FFN grid sizes
    const int par = __ldcg(p.ep_par);  // flipped by the route: this step's counts at [par ^ 1]
    const int* cnt = p.ep_cnt_l + (par ^ 1) * p.ep_El;
    const int per = (p.ep_El + (int)gridDim.x - 1) / (int)gridDim.x;
    const int e0 = blockIdx.x * per, e1 = min(p.ep_El, e0 + per);
    for (int i = threadIdx.x; i < p.ep_P * (e1 - e0); i += blockDim.x) {
      const int dst = i / (e1 - e0), e = e0 + i - dst * (e1 - e0);
      reinterpret_cast<int*>(p.ep_base[dst] + p.ep_off_hits)[p.ep_e0 + e] = __ldcg(cnt + e);
    }
    __syncthreads();
    if (threadIdx.x == 0 && p.ep_P > 1) {  // world 1: the final kernel's wait on this grid
      fence_release_sys();
      for (int dst = 0; dst < p.ep_P; ++dst)
        red_relaxed_sys_add_u32(reinterpret_cast<unsigned*>(p.ep_base[dst] + p.ep_off_ctr) + 2 + par, 1u);
    }
  }
}

}  // namespace tide
