"""Pins for the CPU oracle (oracle/tide_oracle.c) against things that are NOT
the oracle: the worked examples SPEC.md prints (tests/golden/), brute force on
tiny inputs, closed forms, textbook formulas evaluated with NumPy, and the
invariants the paper fixes (Sum hits = N*k, lossless, tau=1 == per-step
refresh, C=E == no offload).  Each test names the oracle part it pins
(O1..O11) and the passage that fixes the expectation.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle
import tidegen as g

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def bf16(a):
    return g.f32_to_bf16_bits(np.asarray(a, np.float32))


def f32(b):
    return g.bf16_bits_to_f32(b).astype(np.float64)


# ------------------------------------------------------------------ O6 / O5
@pytest.mark.parametrize("ex", GOLD["select_top_b"], ids=lambda e: e["cite"])
def test_placement_spec_examples(ex):
    """O6 vs SPEC's printed top-B examples."""
    h = np.array(ex["hits"], np.int32)
    p = oracle.placement(h, ex["B"], refresh=True)
    assert sorted(np.nonzero(p)[0].tolist()) == ex["expect"]


@pytest.mark.parametrize("ex", GOLD["refresh_flags"], ids=lambda e: e["cite"])
def test_refresh_flags_spec(ex):
    """O5 vs S:247 / S:249 (Alg. 1 line 2)."""
    assert [oracle.is_refresh(t, ex["interval"]) for t in range(ex["T"])] == ex["expect"]


def test_promotions_evictions_spec():
    """O10 promotions/evictions are set differences."""
    ex = GOLD["promotions_evictions"][0]
    E = ex["E"]
    old = np.zeros(E, np.uint8)
    old[ex["old"]] = 1
    new = np.zeros(E, np.uint8)
    new[ex["new"]] = 1
    hits = np.zeros(E, np.int32)
    io = oracle.io_step(hits, old, new, old.copy(), lazy=True)
    assert io["promotions"] == len(ex["promotions"]) and io["evictions"] == len(ex["evictions"])


def test_route_tokens_spec():
    """O7 bucket sizes vs S:259."""
    ex = GOLD["route_tokens"][0]
    topk = np.array(ex["topk"], np.int32)
    pl = np.zeros(ex["E"], np.uint8)
    pl[ex["resident"]] = 1
    order, offsets, pos = oracle.buckets(topk, pl)
    n_res = int(pl.sum())
    assert offsets[n_res] == ex["resident_pairs"]
    assert offsets[-1] - offsets[n_res] == ex["nonresident_pairs"]


def _brute_top_c(hits, C):
    """Brute force: the C-subset maximising Sum hits; among maximisers
    the lexicographically smallest id tuple."""
    E = len(hits)
    best, best_set = None, None
    for comb in itertools.combinations(range(E), C):  # lexicographic order
        s = sum(int(hits[e]) for e in comb)
        if best is None or s > best:
            best, best_set = s, comb
    return set(best_set)


@pytest.mark.parametrize("seed", range(40))
def test_placement_brute_force(seed):
    """O6 == exhaustive search over all C-subsets on tiny layers (E <= 10)."""
    rng = np.random.default_rng(seed)
    E = int(rng.integers(2, 11))
    C = int(rng.integers(1, E + 1))
    hits = rng.integers(0, 5, E).astype(np.int32)
    p = oracle.placement(hits, C, refresh=True)
    assert set(np.nonzero(p)[0].tolist()) == _brute_top_c(hits, C)
    assert int(p.sum()) == C


def test_placement_skipped_step_keeps_input():
    """skipped steps keep the placement; S:242 refresh only at t%tau==0."""
    pin = np.array([0, 1, 1, 0, 1], np.uint8)
    p = oracle.placement(np.array([9, 0, 0, 9, 0], np.int32), 3, refresh=False, placement_in=pin)
    assert (p == pin).all()


def test_capacity_equals_E_is_all_resident():
    """C = E -> everything resident (no offload, BASELINE north_star)."""
    h = np.random.default_rng(0).integers(0, 7, 32).astype(np.int32)
    assert oracle.placement(h, 32, refresh=True).all()


# ------------------------------------------------------------------ O2
@pytest.mark.parametrize("seed", range(20))
def test_topk_against_full_sort(seed):
    """O2 == Python's full stable sort by (logit desc, id asc) -- with ties."""
    rng = np.random.default_rng(seed)
    N, E = 7, int(rng.integers(2, 40))
    k = int(rng.integers(1, E + 1))
    logits = rng.integers(-3, 4, (N, E)).astype(np.float64)  # many exact ties
    t = oracle.topk(logits, k)
    for n in range(N):
        ref = sorted(range(E), key=lambda e: (-logits[n, e], e))[:k]
        assert t[n].tolist() == ref


def test_topk_distinct_and_in_range():
    rng = np.random.default_rng(3)
    t = oracle.topk(rng.standard_normal((50, 64)), 8)
    assert all(len(set(r)) == 8 for r in t.tolist()) and t.min() >= 0 and t.max() < 64


# ------------------------------------------------------------------ O1 + O3
def test_zero_router_gives_lowest_ids_uniform_gates():
    """Wr = 0 -> all logits 0 -> top-k = {0..k-1} by tie-break, gates 1/k."""
    N, E, H, k = 5, 16, 32, 4
    x = bf16(np.random.default_rng(1).standard_normal((N, H)))
    wr = bf16(np.zeros((E, H)))
    lg = oracle.router_logits(x, wr)
    assert (lg == 0).all()
    t = oracle.topk(lg, k)
    assert (t == np.arange(k)).all()
    assert np.allclose(oracle.gates(lg, t, True), 1.0 / k, rtol=0, atol=1e-15)
    assert np.allclose(oracle.gates(lg, t, False), 1.0 / E, rtol=0, atol=1e-15)


def test_one_hot_router_logits_are_known_constants():
    """Wr[e] = c_e * onehot(h=0), x[:,0] = 1 -> logits[n,e] = c_e exactly."""
    N, E, H = 3, 8, 16
    x = np.random.default_rng(2).standard_normal((N, H)).astype(np.float32)
    x[:, 0] = 1.0
    c = np.array([0.5, -1.0, 2.0, 0.25, 3.0, -2.0, 1.5, 0.0], np.float32)
    wr = np.zeros((E, H), np.float32)
    wr[:, 0] = c
    lg = oracle.router_logits(x, wr)
    assert (lg == c[None, :]).all()
    assert oracle.topk(lg, 3)[0].tolist() == [4, 2, 6]


def test_logits_match_numpy_fp64_matmul():
    """O1 vs an independent library routine (NumPy fp64 matmul on the exact
    bf16 values); only the summation order differs -> ~1e-15 relative."""
    rng = np.random.default_rng(4)
    x = bf16(rng.standard_normal((6, 256)))
    wr = bf16(rng.uniform(-0.1, 0.1, (32, 256)))
    ref = f32(x) @ f32(wr).T
    assert np.allclose(oracle.router_logits(x, wr), ref, rtol=1e-13, atol=1e-14)


def test_gates_closed_forms():
    """O3: renormalised gates == softmax over the k selected logits; with
    k=2 that is a sigmoid of the logit gap; p sums to 1 over all E."""
    rng = np.random.default_rng(5)
    lg = rng.standard_normal((9, 12)) * 3
    t = oracle.topk(lg, 2)
    gn = oracle.gates(lg, t, True)
    l1 = np.take_along_axis(lg, t, 1)
    assert np.allclose(gn[:, 0], 1 / (1 + np.exp(-(l1[:, 0] - l1[:, 1]))), atol=1e-14)
    assert np.allclose(gn.sum(1), 1.0, atol=1e-14)
    t_all = oracle.topk(lg, 12)
    assert np.allclose(oracle.gates(lg, t_all, False).sum(1), 1.0, atol=1e-14)
    p = np.exp(lg) / np.exp(lg).sum(1, keepdims=True)
    assert np.allclose(oracle.gates(lg, t, False), np.take_along_axis(p, t, 1), atol=1e-15)


# ------------------------------------------------------------------ O4
def test_hits_sum_and_bound():
    """O4: Sum hits = N*k; each hits[e] <= N (a token selects e once)."""
    rng = np.random.default_rng(6)
    lg = rng.standard_normal((33, 64))
    t = oracle.topk(lg, 8)
    h = oracle.hits(t, 64)
    assert h.sum() == 33 * 8 and h.max() <= 33
    assert (h == np.bincount(t.ravel(), minlength=64)).all()


# ------------------------------------------------------------------ O7
@pytest.mark.parametrize("seed", range(10))
def test_buckets_are_a_canonical_permutation(seed):
    """O7: pos is a bijection onto [0, N*k); each expert owns a contiguous
    run of rows in ascending token order; resident experts come first."""
    rng = np.random.default_rng(seed)
    N, E, k = int(rng.integers(1, 40)), 24, 3
    t = oracle.topk(rng.standard_normal((N, E)), k)
    pl = g.random_placement(E, int(rng.integers(1, E + 1)), seed)
    order, offsets, pos = oracle.buckets(t, pl)
    assert sorted(pos.ravel().tolist()) == list(range(N * k))
    res = [e for e in range(E) if pl[e]]
    assert order.tolist() == res + [e for e in range(E) if not pl[e]]
    h = np.bincount(t.ravel(), minlength=E)
    for i, e in enumerate(order):
        rows = [(pos[n, j], n) for n in range(N) for j in range(k) if t[n, j] == e]
        rows.sort()
        assert [r for r, _ in rows] == list(range(offsets[i], offsets[i] + h[e]))
        assert [n for _, n in rows] == sorted(n for _, n in rows)


# ------------------------------------------------------------------ O8
def _np_swiglu(x, wg, wu, wd):
    u, v = wg @ x, wu @ x
    return wd @ (u * (1 / (1 + np.exp(-u))) * v)


def test_swiglu_matches_textbook_numpy():
    """O8 vs the textbook SwiGLU MLP written with NumPy fp64 matmuls."""
    rng = np.random.default_rng(7)
    H, F = 48, 40
    wg, wu = bf16(rng.uniform(-.3, .3, (F, H))), bf16(rng.uniform(-.3, .3, (F, H)))
    wd = bf16(rng.uniform(-.3, .3, (H, F)))
    x = f32(bf16(rng.standard_normal(H)))
    ref = _np_swiglu(x, f32(wg), f32(wu), f32(wd))
    assert np.allclose(oracle.swiglu(x, wg, wu, wd), ref, rtol=1e-12, atol=1e-13)


def test_swiglu_zero_gate_is_zero():
    """silu(0) = 0 -> Wg = 0 gives y = 0 exactly."""
    rng = np.random.default_rng(8)
    H, F = 16, 8
    y = oracle.swiglu(rng.standard_normal(H), np.zeros((F, H), np.float32),
                      rng.standard_normal((F, H)).astype(np.float32),
                      rng.standard_normal((H, F)).astype(np.float32))
    assert (y == 0).all()


# ------------------------------------------------------------------ O9 / step
def _tiny_layer(seed, E=6, H=32, F=24, shared=False, dtype="bf16"):
    shp = g.Shape("t", E, 2, H, F, 1, 5, steps=4, dtype=dtype, shared_expert=shared)
    lt = g.layer_np(shp, seed)
    return shp, oracle.Layer(lt.wr, lt.wg, lt.wu, lt.wd, lt.shared)


@pytest.mark.parametrize("shared", [False, True])
def test_step_equals_dense_all_experts_moe(shared):
    """O9 == dense form out[n] = Sum_{e<E} G[n,e] FFN_e(x_n) (+ shared) with G
    zero off-selection, evaluated independently with NumPy (the
    method reaches the dense all-experts result)."""
    shp, L = _tiny_layer(11, shared=shared)
    x = g.block_hidden_np(shp, 11)[0]
    E, k = shp.num_experts, shp.top_k
    r = oracle.moe_step(L, x, k, np.zeros(E, np.uint8), 0, 1, 3)
    assert r.status == 0
    X = f32(x)
    logits = X @ f32(L.wr).T
    G = np.zeros_like(logits)
    for n in range(X.shape[0]):
        sel = sorted(range(E), key=lambda e: (-logits[n, e], e))[:k]
        z = np.exp(logits[n, sel] - logits[n, sel].max())
        G[n, sel] = z / z.sum()
    dense = np.zeros_like(X)
    for n in range(X.shape[0]):
        for e in range(E):
            if G[n, e]:
                dense[n] += G[n, e] * _np_swiglu(X[n], f32(L.wg[e]), f32(L.wu[e]), f32(L.wd[e]))
        if shared:
            dense[n] += _np_swiglu(X[n], *(f32(a) for a in L.shared))
    assert np.allclose(r.out, dense, rtol=1e-11, atol=1e-12)


def test_single_expert_reduces_to_dense_swiglu():
    """E = k = 1: the MoE layer is one textbook SwiGLU MLP with gate 1."""
    shp, L = _tiny_layer(12, E=1)
    x = g.block_hidden_np(shp, 12)[0]
    r = oracle.moe_step(L, x, 1, np.zeros(1, np.uint8), 0, 1, 1)
    ref = np.stack([_np_swiglu(xx, f32(L.wg[0]), f32(L.wu[0]), f32(L.wd[0])) for xx in f32(x)])
    assert np.allclose(r.gates, 1.0) and np.allclose(r.out, ref, rtol=1e-12, atol=1e-13)


def test_identical_experts_with_renorm_equal_one_ffn():
    """All experts identical + renormalised gates -> out = FFN(x)."""
    shp, L = _tiny_layer(13)
    for e in range(1, shp.num_experts):
        L.wg[e], L.wu[e], L.wd[e] = L.wg[0], L.wu[0], L.wd[0]
    x = g.block_hidden_np(shp, 13)[0]
    r = oracle.moe_step(L, x, 2, np.zeros(shp.num_experts, np.uint8), 0, 1, 2)
    ref = np.stack([_np_swiglu(xx, f32(L.wg[0]), f32(L.wu[0]), f32(L.wd[0])) for xx in f32(x)])
    assert np.allclose(r.out, ref, rtol=1e-12, atol=1e-12)


def test_lossless_across_placement_interval_capacity():
    """outputs do not depend on placement, interval or capacity."""
    shp, L = _tiny_layer(14)
    x = g.block_hidden_np(shp, 14)[0]
    E = shp.num_experts
    base = oracle.moe_step(L, x, 2, np.zeros(E, np.uint8), 0, 1, E).out
    for cap, itv, step in [(1, 1, 0), (2, 3, 1), (3, 2, 3), (E, 5, 2)]:
        pin = g.random_placement(E, cap, cap)
        r = oracle.moe_step(L, x, 2, pin, step, itv, cap)
        assert r.status == 0 and (r.out == base).all()


def test_nonrefresh_placement_over_capacity_is_rejected():
    """S:49, S:263 budget safety: a skipped step with |placement| > C errors."""
    shp, L = _tiny_layer(15)
    x = g.block_hidden_np(shp, 15)[0]
    r = oracle.moe_step(L, x, 2, np.ones(shp.num_experts, np.uint8), 1, 2, 2)
    assert r.status == 3


def test_token_mask_restricts_ffn_only():
    shp, L = _tiny_layer(16)
    x = g.block_hidden_np(shp, 16)[0]
    full = oracle.moe_step(L, x, 2, np.zeros(6, np.uint8), 0, 1, 6)
    m = np.array([1, 0, 1, 0, 0], np.uint8)
    part = oracle.moe_step(L, x, 2, np.zeros(6, np.uint8), 0, 1, 6, token_mask=m)
    assert (part.out[m == 1] == full.out[m == 1]).all() and (part.out[m == 0] == 0).all()
    assert (part.hits == full.hits).all()


# ------------------------------------------------------------------ schedule
def _per_step_policy(hits_seq, C):
    """Mixtral-Offload style per-step refresh, coded independently:
    every step, resident = first C of ids sorted by (-hits, id)."""
    out = []
    for h in hits_seq:
        p = np.zeros(len(h), np.uint8)
        p[np.lexsort((np.arange(len(h)), -np.asarray(h)))[:C]] = 1
        out.append(p)
    return out


def test_interval_one_equals_per_step_refresh():
    """S:249 / P:237: tau = 1 recovers the per-step (full-refresh) baseline."""
    shp = g.TOY
    lt = g.layer_np(shp, 21)
    L = oracle.Layer(lt.wr, lt.wg, lt.wu, lt.wd)
    xs = g.block_hidden_np(shp, 21)
    p = np.zeros(shp.num_experts, np.uint8)
    got, hs = [], []
    for t in range(shp.steps):
        r = oracle.moe_step(L, xs[t], shp.top_k, p, t, 1, shp.capacity)
        got.append(r.placement)
        hs.append(r.hits)
        p = r.placement
    for a, b in zip(got, _per_step_policy(hs, shp.capacity)):
        assert (a == b).all()


def test_interval_schedule_refreshes_only_on_cadence():
    """Alg. 1: placement changes only at t % tau == 0 and the
    resident set never exceeds C."""
    shp = g.TOY
    lt = g.layer_np(shp, 22)
    L = oracle.Layer(lt.wr, lt.wg, lt.wu, lt.wd)
    xs = g.block_hidden_np(shp, 22, iid=True)
    p = np.zeros(shp.num_experts, np.uint8)
    for t in range(shp.steps):
        r = oracle.moe_step(L, xs[t], shp.top_k, p, t, 3, shp.capacity)
        if t % 3:
            assert (r.placement == p).all()
        assert r.placement.sum() <= shp.capacity
        p = r.placement


# ------------------------------------------------------------------ O10
def test_io_model_invariants():
    """O10: migrations per refresh <= C; a static placement after
    warm-up copies nothing when every hit expert is resident; C = E lazy ->
    each expert copied at most once over a block (no offload thereafter)."""
    rng = np.random.default_rng(30)
    E, C = 32, 8
    loaded = np.zeros(E, np.uint8)
    p = np.zeros(E, np.uint8)
    for t in range(20):
        h = np.bincount(rng.choice(E, 12), minlength=E).astype(np.int32)
        po = oracle.placement(h, C, refresh=(t % 2 == 0), placement_in=p)
        io = oracle.io_step(h, p, po, loaded, lazy=False)
        assert io["promotions"] <= C and io["evictions"] <= C
        assert loaded.sum() <= C and not (loaded & (1 - po)).any()
        assert io["resident_pairs"] + io["nonresident_pairs"] == h.sum()
        p = po
    loaded = np.zeros(E, np.uint8)
    total = 0
    allp = np.ones(E, np.uint8)
    for t in range(10):
        h = np.bincount(rng.choice(E, 12), minlength=E).astype(np.int32)
        total += oracle.io_step(h, allp, allp, loaded, lazy=True)["copies"]
    assert total <= E and total == int(loaded.sum())
    h = np.ones(E, np.int32)
    assert oracle.io_step(h, allp, allp, np.ones(E, np.uint8), lazy=True)["copies"] == 0


def test_io_model_streams_nonresident_hits_every_step():
    """R-13: a hit non-resident expert is copied (staged) on every step it is
    hit, and is not retained."""
    E = 4
    p = np.array([1, 0, 0, 0], np.uint8)
    loaded = np.array([1, 0, 0, 0], np.uint8)
    h = np.array([1, 2, 0, 1], np.int32)
    for _ in range(3):
        io = oracle.io_step(h, p, p, loaded, lazy=True)
        assert io["experts_streamed"] == 2 and io["copies"] == 2
        assert loaded.tolist() == [1, 0, 0, 0]


# ------------------------------------------------------------------ O11
@pytest.mark.parametrize("P", [1, 2, 3])
def test_ep_emulation_equals_single_device(P):
    """O11: EP moves bytes, not math -> hits identical, out equal up to fp64
    summation order, per-rank placement = brute-force top-C_r of the rank's
    experts by global hits."""
    shp, L = _tiny_layer(40, E=6)
    x = g.block_hidden_np(shp, 40)[0]
    E, k = 6, 2
    single = oracle.moe_step(L, x, k, np.zeros(E, np.uint8), 0, 1, E)
    cr = 1
    t, h, pout, out = oracle.ep_step(L, P, x, k, np.zeros(E, np.uint8), 0, 1, cr)
    assert (t == single.topk_idx).all() and (h == single.hits).all()
    assert np.allclose(out, single.out, rtol=1e-13, atol=1e-14)
    El = E // P
    for r in range(P):
        want = {r * El + e for e in _brute_top_c(h[r * El:(r + 1) * El], cr)}
        assert set(np.nonzero(pout[r * El:(r + 1) * El])[0] + r * El) == want


# ------------------------------------------------------------------ O10 eviction timing (R-12)
def test_io_eviction_timing_hand_worked():
    """O10 vs a hand-worked three-step example (tests/golden/io_eviction_timing.json, DESIGN
    R-12/R-13): an expert evicted at a refresh is still served from HBM in that step, so it is
    not streamed; the alternative rule (evict before counting) would stream it."""
    ex = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                     "io_eviction_timing.json")))
    E = ex["E"]
    loaded = np.zeros(E, np.uint8)
    for st in ex["steps"]:
        h = np.array(st["hits"], np.int32)
        pin = np.array(st["placement_in"], np.uint8)
        po = oracle.placement(h, ex["capacity"], st["refresh"], pin)
        assert po.tolist() == st["placement_out"], st["step"]
        io = oracle.io_step(h, pin, po, loaded, lazy=bool(ex["lazy"]))
        assert io == st["expect"], (st["step"], io)
        assert loaded.tolist() == st["loaded_after"], st["step"]


# ------------------------------------------------------------------ threading
def test_threads_bit_identical():
    """The oracle's per-token loops run on host threads (bench.py cpu_baseline on nproc cores);
    a token's arithmetic never crosses threads, so 1 and 4 threads give identical bits for the
    whole step (O1..O9) and the EP emulation (O11)."""
    shp, L = _tiny_layer(77, E=8, H=64, F=64, shared=True)
    x = g.block_hidden_np(shp, 77, tokens=23)[0]
    E, k = shp.num_experts, shp.top_k
    res = []
    for nt in (1, 4):
        oracle.set_threads(nt)
        assert oracle.get_threads() == nt
        r = oracle.moe_step(L, x, k, np.zeros(E, np.uint8), 0, 1, 3)
        ep = oracle.ep_step(L, 2, x, k, np.zeros(E, np.uint8), 0, 1, 2)
        res.append((r, ep))
    oracle.set_threads(os.cpu_count() or 1)
    (a, ea), (b, eb) = res
    assert a.logits.tobytes() == b.logits.tobytes()
    assert a.out.tobytes() == b.out.tobytes()
    assert (a.topk_idx == b.topk_idx).all() and (a.pos == b.pos).all()
    assert ea[3].tobytes() == eb[3].tobytes()
