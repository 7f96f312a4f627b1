"""NEXT-4 on the GPU: tide_trace_stats (cosine similarity matrix, unique experts, Eq. 4
drift) on hit counts captured from the library's own layer-steps, exact against the
oracle, and the captured routing reproduces the paper's statistics."""
import numpy as np
import pytest
import torch

import oracle
import tidegen as g
from tests._util import DeviceLayer, desc_for

pytestmark = pytest.mark.gpu


def test_trace_stats_random_counts_exact():
    from paper_2605_20179_b200 import tide
    rng = np.random.default_rng(3)
    T, E, B = 9, 96, 20
    C = rng.integers(0, 6, (T, E)).astype(np.int32)
    C[4] = 0  # an all-zero step: similarity 0
    sim, uq, dr = tide.trace_stats(torch.from_numpy(C).cuda(), B)
    torch.cuda.synchronize()
    sim, uq, dr = sim.cpu().numpy(), uq.cpu().numpy(), dr.cpu().numpy()
    for s in range(T):
        assert uq[s] == oracle.unique(C[s])
        for t in range(T):
            assert sim[s, t] == oracle.cosine(C[s], C[t])
    for t in range(1, T):
        assert dr[t - 1] == oracle.drift(C[t - 1], C[t], B)


def test_trace_stats_on_captured_routing():
    from paper_2605_20179_b200 import tide
    shape = g.Shape("mini_r", 256, 8, 2048, 64, 1, 32, steps=32, dtype="bf16")  # router-sized
    layer = DeviceLayer(shape, 7)
    ctx = tide.Context(desc_for(shape), 256)
    xs = g.block_hidden_np(shape, 7)
    counts = torch.empty(shape.steps, 256, dtype=torch.int32, device="cuda")
    pl = torch.zeros(256, dtype=torch.uint8, device="cuda")
    for t in range(shape.steps):
        ctx.moe_step(g.np_to_torch(xs[t], "cuda"), layer.router, **layer.weights(), placement=pl,
                     step=t, interval=1, hit_counts=counts[t])
    sim, uq, dr = tide.trace_stats(counts, 64)
    torch.cuda.synchronize()
    C = counts.cpu().numpy()
    sim = sim.cpu().numpy()
    adj = np.mean([sim[t, t + 1] for t in range(31)])
    lag5 = np.mean([sim[t, t + 5] for t in range(27)])
    assert 0.975 <= adj <= 0.995 and lag5 > 0.95, (adj, lag5)
    assert (uq.cpu().numpy() == [oracle.unique(c) for c in C]).all()
    assert np.allclose(dr.cpu().numpy(), [oracle.drift(C[t - 1], C[t], 64) for t in range(1, 32)])


@pytest.mark.parametrize("counter,incumbent", [("window", False), ("cumulative", True),
                                               ("current", True), ("window", True)])
def test_counter_modes_schedule(counter, incumbent):
    """NEXT-1 on the GPU: placement' at every step equals the oracle's counter reading +
    incumbent-aware top-C, fed the GPU's own hits (outputs unchanged: lossless)."""
    from paper_2605_20179_b200 import tide
    shape = g.Shape("cm", 48, 4, 128, 64, 1, 16, steps=10, dtype="bf16")
    layer = DeviceLayer(shape, 61)
    E, C, tau = 48, 12, 3
    desc = tide.make_desc(E, 4, 128, 64, 16, counter=counter, incumbent_ties=incumbent)
    ctx = tide.Context(desc, C)
    base = tide.Context(desc_for(shape), C)
    xs = g.block_hidden_np(shape, 61)
    mode = {"current": 0, "window": 1, "cumulative": 2}[counter]
    acc = np.zeros(E, np.int32)
    p = np.zeros(E, np.uint8)
    p[:C] = 1
    for blk in range(2):
        for t in range(shape.steps):
            x = g.np_to_torch(xs[t], "cuda")
            r = ctx.moe_step(x, layer.router, **layer.weights(),
                             placement=torch.from_numpy(p.copy()).cuda(), step=t, interval=tau)
            r0 = base.moe_step(x, layer.router, **layer.weights(),
                               placement=torch.from_numpy(p.copy()).cuda(), step=t, interval=tau)
            torch.cuda.synchronize()
            hits = r.hit_counts.cpu().numpy()
            key = oracle.counter_key(mode, t, hits, acc)
            want = oracle.placement_ex(key, C, t % tau == 0, incumbent, p)
            oracle.counter_update(mode, t, t % tau == 0, hits, acc)
            assert (r.placement.cpu().numpy() == want).all(), (blk, t)
            assert torch.equal(r.out.view(torch.int16), r0.out.view(torch.int16))
            p = want


def test_h2d_prefetch_is_bitwise_neutral_and_used():
    """NEXT-3 H2D prefetch (host_master): a 3-layer ring at C < E where each layer's step
    copies the next layer's predicted streamed experts into that layer's prefetch slots.
    Outputs, hits and placements are bitwise those of the same ring without prefetch; the
    prefetched experts are used (fewer H2D copies on the steps after the first), and every
    prefetch copy is counted in the stats."""
    from paper_2605_20179_b200 import tide
    shape = g.Shape("pfh", 32, 4, 256, 256, 1, 24, steps=6, dtype="bf16", shared_expert=True)
    E, C = shape.num_experts, 6
    layers = [DeviceLayer(shape, 90 + l, host_master=True) for l in range(3)]
    xs = [g.block_hidden_np(shape, 90 + l) for l in range(3)]

    def run(prefetch):
        ctxs = [tide.Context(desc_for(shape), C, 4) for _ in layers]
        if prefetch:
            for l, c in enumerate(ctxs):
                c.set_prefetch(ctxs[(l + 1) % 3], None, 4 * shape.expert_bytes)
        pls = [torch.zeros(E, dtype=torch.uint8, device="cuda") for _ in layers]
        res, copies = [], 0
        for t in range(shape.steps):
            for l, (L, c) in enumerate(zip(layers, ctxs)):
                r = c.moe_step(g.np_to_torch(xs[l][t], "cuda"), L.router, **L.weights("host_master"),
                               placement=pls[l], step=t, interval=2, placement_out=pls[l], stats=True)
                torch.cuda.synchronize()
                res.append((r.out.view(torch.int16).cpu().numpy().copy(),
                            r.hit_counts.cpu().numpy().copy(), r.placement.cpu().numpy().copy()))
                copies += r.stats["copies"]
        return res, copies

    base, c0 = run(False)
    got, c1 = run(True)
    for (a, ha, pa), (b, hb, pb) in zip(base, got):
        assert (a == b).all() and (ha == hb).all() and (pa == pb).all()
    assert c1 > 0 and c0 > 0


@pytest.mark.parametrize("tau,lazy", [(1, False), (3, False), (4, True), (8, False)])
def test_interval_replay_predicts_measured_copies(tau, lazy):
    """NEXT-2 replay (R-24): the expert copies the host_master step issued over a block (the
    second of two back-to-back blocks, placement carried across) equal the replay of the
    GPU's own captured routing exactly, per step."""
    from paper_2605_20179_b200 import tide
    shape = g.Shape("rp", 64, 4, 256, 128, 1, 48, steps=12, dtype="bf16", shared_expert=True)
    E, C = shape.num_experts, 20
    layer = DeviceLayer(shape, 71, host_master=True)
    ctx = tide.Context(tide.make_desc(E, 4, 256, 128, 48, shared_expert=True, lazy_promote=lazy), C, 8)
    xs = g.block_hidden_np(shape, 71)
    pl = torch.zeros(E, dtype=torch.uint8, device="cuda")
    counts = np.zeros((shape.steps, E), np.int32)
    measured = np.zeros(shape.steps, np.int64)
    for blk in range(2):
        for t in range(shape.steps):
            r = ctx.moe_step(g.np_to_torch(xs[t], "cuda"), layer.router, **layer.weights("host_master"),
                             placement=pl, step=t, interval=tau, placement_out=pl, stats=True)
            torch.cuda.synchronize()
            if blk == 1:
                counts[t] = r.hit_counts.cpu().numpy()
                measured[t] = r.stats["copies"]
    tot, per = tide.interval_replay(counts, C, tau, lazy, 2)
    assert per.tolist() == measured.tolist() and tot == measured.sum()
    assert oracle.interval_replay(counts, C, tau, lazy, 2)[1].tolist() == measured.tolist()
