"""NEXT-2 (refresh-interval model, Eq. 4-7) and NEXT-4 (routing-trace analytics):
oracle pins (SPEC worked examples, limits, monotonicity) and the library's host
optimizer against the oracle (no GPU needed); the GPU analytics kernel is checked in
tests/test_gpu_next.py."""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


@pytest.mark.parametrize("ex", GOLD["eq5_migrations"], ids=lambda e: f"tau{e['tau']}")
def test_eq5_spec_examples(ex):
    """Eq. 5 vs S:324-326: 204.8 at tau=1 (= B*T*d) and 176.0768 at tau=4."""
    got = oracle.migration_cost(ex["tau"], ex["B"], ex["T"], ex["d"], 1.0)
    assert got == pytest.approx(ex["expect"], rel=1e-12)


@pytest.mark.parametrize("ex", GOLD["miss_fraction"], ids=lambda e: e["cite"])
def test_miss_fraction_spec_examples(ex):
    assert oracle.miss_fraction(ex["tau"], ex["d"]) == pytest.approx(ex["expect"], abs=1e-9)


def test_interval_model_limits_and_monotonicity():
    """tau=1 recovers B*T*d; d=1 gives exactly B*T/tau (the 1/tau scaling);
    d=0 costs nothing; migrations non-increasing and misses non-decreasing in tau
    (Fig. 4a)."""
    B, T = 48, 32
    for d in (0.0, 0.05, 0.3, 1.0):
        io = [oracle.migration_cost(t, B, T, d, 1.0) for t in range(1, T)]
        ms = [oracle.miss_cost(t, B, T, d, 1.0) for t in range(1, T)]
        assert all(a >= b - 1e-9 for a, b in zip(io, io[1:]))
        assert all(a <= b + 1e-9 for a, b in zip(ms, ms[1:]))
        assert io[0] == pytest.approx(B * T * d, abs=1e-9)
        if d == 1.0:
            assert all(io[t - 1] == pytest.approx(B * T / t) for t in range(1, T))
        if d == 0.0:
            assert max(io) == 0 and max(ms) == 0


def test_optimizer_limits():
    """d=0 -> tau*=1 (tie -> smallest); c_miss=0 with d>0 -> tau*=T-1.
    With c_miss = c_io (B200: a miss streams the expert like a migration, R-13) the
    per-step refresh tau=1 is optimal for every d (SURVEY 8(d) finding)."""
    assert oracle.optimize_tau(32, 64, 0.0, 1.0, 1.0)[0] == 1
    assert oracle.optimize_tau(32, 64, 0.1, 1.0, 0.0)[0] == 31
    for d in (0.01, 0.1, 0.5):
        assert oracle.optimize_tau(32, 64, d, 1.0, 1.0)[0] == 1
    tau, curve = oracle.optimize_tau(20, 16, 0.2, 1.0, 0.3)
    assert tau == 1 + int(np.argmin(curve))


@pytest.mark.parametrize("seed", range(12))
def test_library_optimizer_matches_oracle(seed):
    """libtide.so's host-side tide_optimize_interval / tide_interval_cost vs the oracle."""
    from paper_2605_20179_b200 import _build
    _build.build()
    from paper_2605_20179_b200 import tide
    rng = np.random.default_rng(seed)
    T, B = int(rng.integers(2, 64)), int(rng.integers(1, 256))
    d, c_io, c_miss = float(rng.uniform(0, 1)), float(rng.uniform(0.1, 5)), float(rng.uniform(0, 5))
    tau, curve = tide.optimize_interval(T, B, d, c_io, c_miss)
    otau, ocurve = oracle.optimize_tau(T, B, d, c_io, c_miss)
    assert tau == otau
    assert np.allclose(curve, ocurve, rtol=1e-12, atol=1e-9)
    for t in (1, max(1, T // 2), T - 1):
        io, ms = tide.interval_cost(T, B, d, c_io, c_miss, t)
        assert io == pytest.approx(oracle.migration_cost(t, B, T, d, c_io), rel=1e-12, abs=1e-12)
        assert ms == pytest.approx(oracle.miss_cost(t, B, T, d, c_miss), rel=1e-12, abs=1e-12)


@pytest.mark.parametrize("ex", GOLD["similarity"], ids=lambda e: e["cite"])
def test_similarity_spec_examples(ex):
    assert oracle.cosine(np.array(ex["a"]), np.array(ex["b"])) == pytest.approx(ex["expect"])


def test_similarity_zero_vector():
    assert oracle.cosine(np.zeros(4, np.int32), np.array([1, 2, 0, 0])) == 0.0


@pytest.mark.parametrize("ex", GOLD["drift"], ids=lambda e: e["cite"])
def test_drift_spec_examples(ex):
    assert oracle.drift(np.array(ex["prev"]), np.array(ex["cur"]), ex["B"]) == ex["expect"]
    assert oracle.drift(np.array(ex["cur"]), np.array(ex["cur"]), ex["B"]) == 0.0


@pytest.mark.parametrize("ex", GOLD["unique"], ids=lambda e: e["cite"])
def test_unique_spec_examples(ex):
    h = oracle.hits(np.array(ex["topk"], np.int32), ex["E"])
    assert oracle.unique(h) == ex["expect"]


def test_generator_matches_paper_routing_statistics():
    """The input recipe (DESIGN 4) reproduces the routing statistics the paper prints:
    mean adjacent-step cosine similarity 0.985, > 0.95 five steps apart,
    and unique experts per step growing within the block (Fig. 2a).  Routing
    by the oracle on the mini-shaped router, 32 tokens x 32 steps."""
    import tidegen as g
    s = g.MINI
    wr = g.router_np(s, 7, 0)
    xs = g.block_hidden_np(s, 7, 0)
    C = np.array([oracle.hits(oracle.topk(oracle.router_logits(xs[t], wr), s.top_k), 256)
                  for t in range(s.steps)])
    adj = np.mean([oracle.cosine(C[t], C[t + 1]) for t in range(s.steps - 1)])
    lag5 = np.mean([oracle.cosine(C[t], C[t + 5]) for t in range(s.steps - 5)])
    u = [oracle.unique(c) for c in C]
    assert 0.975 <= adj <= 0.995, adj
    assert lag5 > 0.95, lag5
    assert np.mean(u[-8:]) > np.mean(u[:8]) + 20


# ------------------------------------------------------------------ NEXT-1
def _brute_incumbent(key, C, inc):
    """Brute force: maximise sum(key); among maximisers maximise |S & incumbents|;
    among those the lexicographically smallest id tuple."""
    import itertools
    best, best_s = None, None
    for comb in itertools.combinations(range(len(key)), C):
        score = (sum(int(key[e]) for e in comb), sum(int(inc[e]) for e in comb))
        if best is None or score > best:
            best, best_s = score, comb
    return set(best_s)


@pytest.mark.parametrize("seed", range(30))
def test_incumbent_tie_break_brute_force(seed):
    rng = np.random.default_rng(seed)
    E = int(rng.integers(2, 10))
    C = int(rng.integers(1, E + 1))
    key = rng.integers(0, 3, E).astype(np.int32)
    inc = (rng.random(E) < 0.5).astype(np.uint8)
    got = oracle.placement_ex(key, C, True, True, inc)
    assert set(np.nonzero(got)[0].tolist()) == _brute_incumbent(key, C, inc)
    plain = oracle.placement_ex(key, C, True, False, inc)
    assert (plain == oracle.placement(key, C, True)).all()


def test_counter_window_and_cumulative_sums():
    """at a refresh the window holds the hits of [t_prev_refresh, t) and is reset;
    the cumulative variant holds everything since step 0; step 0 ranks by its own
    hits (OracleStep0 cold start); mode 0 is the current step (R-5)."""
    rng = np.random.default_rng(1)
    E, tau = 6, 2
    h = [rng.integers(0, 5, E).astype(np.int32) for _ in range(5)]
    for mode in (0, 1, 2):
        acc = np.zeros(E, np.int32)
        keys = []
        for t in range(5):
            keys.append(oracle.counter_key(mode, t, h[t], acc))
            oracle.counter_update(mode, t, t % tau == 0, h[t], acc)
        assert (keys[0] == h[0]).all()
        if mode == 0:
            assert all((keys[t] == h[t]).all() for t in range(5))
        if mode == 1:
            assert (keys[2] == h[0] + h[1]).all() and (keys[4] == h[2] + h[3]).all()
            assert (acc == h[4]).all()
        if mode == 2:
            assert (keys[2] == h[0] + h[1]).all() and (keys[4] == h[0] + h[1] + h[2] + h[3]).all()
            assert (acc == sum(h)).all()


# ------------------------------------------------------------------ NEXT-2 on B200 (trace model)
def test_interval_trace_model_hand_worked():
    """Oracle and library vs the hand-worked example (tests/golden/interval_trace_example.json)."""
    from paper_2605_20179_b200 import _build
    _build.build()
    from paper_2605_20179_b200 import tide
    ex = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                     "interval_trace_example.json")))
    c = np.array(ex["counts"], np.int32)
    T = c.shape[0]
    for miss, mig in (oracle.interval_profile(c, ex["B"]), tide.interval_profile(c, ex["B"])):
        assert np.allclose(miss, ex["miss_lag"], rtol=0, atol=1e-15)
        assert np.allclose(mig, ex["mig_lag"], rtol=0, atol=1e-15)
        for tau, want in ex["copies"].items():
            assert oracle.interval_copies_trace(T, int(tau), miss, mig) == pytest.approx(want, abs=1e-12)
            cp, cost = tide.interval_cost_trace(T, 2.0, 0.5, miss, mig, int(tau))
            assert cp == pytest.approx(want, abs=1e-12) and cost == pytest.approx(2 * want + T * 0.5)
        assert tide.optimize_interval_trace(T, 1.0, 0.0, miss, mig)[0] == ex["tau_star"]


def test_interval_trace_model_invariants():
    """A constant trace never migrates and misses the same experts at every lag (copies do not
    depend on tau, so tau* = 1 by the tie rule); B = E never misses or migrates."""
    rng = np.random.default_rng(5)
    row = rng.integers(0, 4, 24).astype(np.int32)
    c = np.tile(row, (10, 1))
    miss, mig = oracle.interval_profile(c, 6)
    assert (mig == 0).all() and np.allclose(miss, miss[0])
    assert miss[0] == ((row > 0).sum() - min(6, (row > 0).sum()))
    copies = [oracle.interval_copies_trace(10, t, miss, mig) for t in range(1, 10)]
    assert np.allclose(copies, 10 * miss[0])
    miss, mig = oracle.interval_profile(rng.integers(0, 3, (8, 24)).astype(np.int32), 24)
    assert (miss == 0).all() and (mig == 0).all()


@pytest.mark.parametrize("seed", range(6))
def test_library_interval_trace_matches_oracle(seed):
    from paper_2605_20179_b200 import tide
    rng = np.random.default_rng(100 + seed)
    T, E = int(rng.integers(2, 40)), int(rng.integers(2, 300))
    B = int(rng.integers(1, E + 1))
    c = rng.poisson(rng.uniform(0.1, 3), (T, E)).astype(np.int32)
    m1, g1 = oracle.interval_profile(c, B)
    m2, g2 = tide.interval_profile(c, B)
    assert (m1 == m2).all() and (g1 == g2).all()
    tau, curve = tide.optimize_interval_trace(T, 1e-4, 1e-5, m2, g2)
    ref = [1e-4 * oracle.interval_copies_trace(T, t, m1, g1) + T * 1e-5 for t in range(1, T)]
    assert np.allclose(curve, ref, rtol=1e-12)
    assert tau == 1 + int(np.argmin(ref))


# ------------------------------------------------------------------ NEXT-2 replay (R-24)
def _replay_golden():
    return json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                       "interval_replay_example.json")))


@pytest.mark.parametrize("ex", _replay_golden()["examples"], ids=lambda e: e["name"])
def test_interval_replay_hand_worked(ex):
    """Oracle and library vs hand-worked replays (tests/golden/interval_replay_example.json):
    eviction timing (R-12), id ties (R-8), eager vs lazy promotion (R-9), cross-block state."""
    from paper_2605_20179_b200 import _build
    _build.build()
    from paper_2605_20179_b200 import tide
    c = np.array(ex["counts"], np.int32)
    for cs in ex["cases"]:
        for fn in (oracle.interval_replay, tide.interval_replay):
            tot, per = fn(c, ex["B"], cs["tau"], bool(cs["lazy"]), cs["passes"])
            assert per.tolist() == cs["per_step"], (fn, cs)
            assert tot == sum(cs["per_step"])


def _top_b(row, B):
    order = np.lexsort((np.arange(row.size), -row.astype(np.int64)))  # hits desc, id asc
    s = np.zeros(row.size, bool)
    s[order[:B]] = True
    return s


@pytest.mark.parametrize("seed", range(4))
def test_interval_replay_tau1_closed_form(seed):
    """tau = 1, eager: the HBM set at a step's start is the previous step's placement, so
    copies(t) = |P_t minus P_{t-1}| + |hit_t minus (P_t union P_{t-1})| (promotions, then the
    streamed experts; R-12 serves a just-evicted expert), P_{-1} = the block's last step in
    the second pass.  Set algebra on numpy lexsort top-B, independent of the step loop."""
    rng = np.random.default_rng(300 + seed)
    T, E = int(rng.integers(2, 20)), int(rng.integers(2, 64))
    B = int(rng.integers(1, E + 1))
    c = rng.poisson(rng.uniform(0.2, 2), (T, E)).astype(np.int32)
    P = [_top_b(c[t], B) for t in range(T)]
    want = []
    for t in range(T):
        prev = P[t - 1]  # t = 0: the previous block's last placement (pass 2)
        want.append(int((P[t] & ~prev).sum() + ((c[t] > 0) & ~(P[t] | prev)).sum()))
    tot, per = oracle.interval_replay(c, B, 1, False, 2)
    assert per.tolist() == want and tot == sum(want)


def test_interval_replay_invariants():
    """B = E: nothing is copied once every expert is in HBM (pass 2 = 0); the cold block
    copies all E experts at step 0 when eager, and each hit expert exactly once (its first
    hit) when lazy.  A constant trace copies only its streamed experts in steady state."""
    rng = np.random.default_rng(11)
    T, E = 9, 40
    c = rng.poisson(0.6, (T, E)).astype(np.int32)
    for tau in (1, 2, 5, 9):
        for lazy in (False, True):
            assert oracle.interval_replay(c, E, tau, lazy, 2)[0] == 0
        tot, per = oracle.interval_replay(c, E, tau, False, 1)
        assert per[0] == E and tot == E
        tot, per = oracle.interval_replay(c, E, tau, True, 1)
        assert tot == int((c > 0).any(axis=0).sum())
    row = rng.integers(0, 4, E).astype(np.int32)
    const = np.tile(row, (T, 1))
    for tau in (1, 3, 9):
        tot, per = oracle.interval_replay(const, 7, tau, False, 2)
        assert (per == (row > 0).sum() - ((row > 0) & _top_b(row, 7)).sum()).all()


@pytest.mark.parametrize("seed", range(6))
def test_library_interval_replay_matches_oracle(seed):
    from paper_2605_20179_b200 import tide
    rng = np.random.default_rng(400 + seed)
    T, E = int(rng.integers(2, 40)), int(rng.integers(2, 300))
    B = int(rng.integers(1, E + 1))
    c = rng.poisson(rng.uniform(0.1, 3), (T, E)).astype(np.int32)
    for tau in sorted({1, 2, int(rng.integers(1, T + 1)), T}):
        for lazy in (False, True):
            for passes in (1, 2, 3):
                a = oracle.interval_replay(c, B, tau, lazy, passes)
                b = tide.interval_replay(c, B, tau, lazy, passes)
                assert a[0] == b[0] and (a[1] == b[1]).all()
    tau, curve = tide.optimize_interval_replay(c, B, 1e-4, 1e-5, T)
    ref = [1e-4 * oracle.interval_replay(c, B, t)[0] + T * 1e-5 for t in range(1, T + 1)]
    assert np.allclose(curve, ref, rtol=1e-12)
    assert tau == 1 + int(np.argmin(ref))
