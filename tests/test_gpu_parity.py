"""GPU parity: libtide.so (through the C ABI) vs the fp64 CPU oracle.

Bar (BASELINE north_star): routing indices, hit counts, placement and the
bucket permutation bit-exact (near-tie tokens with fp64 logit gaps < 1e-6 are
flagged and then the oracle's downstream stages take the GPU's routing);
outputs within max relative error 2e-2 (R-15).
"""
import numpy as np
import pytest
import torch

import oracle
import tidegen as g
from tests._util import (OUT_TOL, DeviceLayer, check_routing, desc_for, rel_err, to_np_f64)

pytestmark = pytest.mark.gpu


def _ctx(shape, capacity, max_tokens=None, norm_topk=True, lazy=False, staging=16):
    from paper_2605_20179_b200 import tide
    return tide.Context(desc_for(shape, max_tokens, norm_topk, lazy), capacity, staging)


def _run_and_check(shape, seed, x_np, layer: DeviceLayer, ctx, placement, step, interval,
                   capacity, mode="device_all", token_mask=None, norm_topk=True):
    E, k = shape.num_experts, shape.top_k
    x = g.np_to_torch(x_np, "cuda")
    pl = torch.from_numpy(placement.copy()).cuda()
    r = ctx.moe_step(x, layer.router, **layer.weights(mode), placement=pl, step=step,
                     interval=interval, capacity=capacity, stats=True, debug=True)
    torch.cuda.synchronize()
    L = layer.oracle_layer(norm_topk)
    ref = oracle.moe_step(L, x_np, k, placement, step, interval, capacity, token_mask=token_mask)
    assert ref.status == 0
    gt = r.debug["topk_idx"].cpu().numpy()
    flagged = check_routing(gt, ref.logits, ref.topk_idx, k)
    # downstream stages: oracle fed the GPU's routing when any token was flagged
    topk = gt if flagged.any() else ref.topk_idx
    hits = oracle.hits(topk, E)
    refresh = oracle.is_refresh(step, interval)
    pl_ref = oracle.placement(hits, capacity, refresh, placement)
    order, offsets, pos = oracle.buckets(topk, pl_ref)
    assert (r.hit_counts.cpu().numpy() == hits).all()
    assert int(r.hit_counts.sum()) == x_np.shape[0] * k
    assert (r.placement.cpu().numpy() == pl_ref).all()
    assert (r.debug["order"].cpu().numpy() == order).all()
    assert (r.debug["offsets"].cpu().numpy() == offsets).all()
    assert (r.debug["pos"].cpu().numpy() == pos).all()
    gates_ref = oracle.gates(ref.logits, topk, norm_topk)
    assert np.abs(r.debug["gates"].cpu().numpy() - gates_ref).max() < 1e-4
    out_ref = ref.out if not flagged.any() else oracle.combine(L, x_np, topk, gates_ref, token_mask)
    out = to_np_f64(r.out)
    sel = slice(None) if token_mask is None else token_mask.astype(bool)
    err = rel_err(out[sel], out_ref[sel])
    assert err < OUT_TOL, f"out rel err {err:.3e}"
    return r, ref, err, flagged


# ------------------------------------------------------------------ toy (fp32, tf32 MMA)
@pytest.mark.parametrize("mode", ["device_all", "host_master"])
def test_toy_schedule(mode):
    """BJ.configs[0]: 16 experts top-2, H=64, F=128, N=8, 8 steps, tau=2, C=4, fp32."""
    shape = g.TOY
    layer = DeviceLayer(shape, 7, host_master=(mode == "host_master"))
    ctx = _ctx(shape, shape.capacity)
    xs = g.block_hidden_np(shape, 7)
    p = np.zeros(shape.num_experts, np.uint8)
    for t in range(shape.steps):
        r, ref, err, _ = _run_and_check(shape, 7, xs[t], layer, ctx, p, t, shape.interval,
                                        shape.capacity, mode)
        p = r.placement.cpu().numpy()


# ------------------------------------------------------------------ bf16 shapes
@pytest.mark.parametrize("shape_name", ["mini", "flash"])
def test_block_layer_parity(shape_name):
    """BJ.configs[1]/[2] layer shapes, block of 32 tokens, C = E: every token's routing,
    hits, placement, permutation and output against the oracle."""
    shape = g.SHAPES[shape_name]
    layer = DeviceLayer(shape, 11)
    ctx = _ctx(shape, shape.num_experts)
    x = g.block_hidden_np(shape, 11, steps=3)[2]
    _run_and_check(shape, 11, x, layer, ctx, np.zeros(shape.num_experts, np.uint8), 0, 1,
                   shape.num_experts)


def test_sweep_batch_parity_capacity_limited():
    """BJ.configs[4]: mini shape, batch of 8 blocks (256 tokens), C = 64 with
    pinned-host serving of non-resident experts; every token's output."""
    shape = g.SWEEP
    layer = DeviceLayer(shape, 12, host_master=True)
    ctx = _ctx(shape, 64)
    x = g.block_hidden_np(shape, 12, steps=1)[0]
    r, *_ = _run_and_check(shape, 12, x, layer, ctx, np.zeros(256, np.uint8), 0, 4, 64,
                           mode="host_master")
    assert r.stats["copies"] > 0 and r.stats["h2d_bytes"] == r.stats["copies"] * shape.expert_bytes


@pytest.mark.parametrize("cap", [64, 217])
def test_flash_capacity_limited_parity(cap):
    """BJ.configs[2] layer shape with pinned-host serving at the paper's budget (C = 64) and
    at C = 217: a refresh step from an empty HBM (promotions + staged chunks), then a
    non-refresh step from its placement (streamed misses only); every token's routing, hits,
    placement, permutation and output against the oracle, and the I/O counters against O10."""
    shape = g.FLASH
    layer = DeviceLayer(shape, 13, host_master=True)
    ctx = _ctx(shape, cap)
    xs = g.block_hidden_np(shape, 13, steps=2)
    pl = np.zeros(shape.num_experts, np.uint8)
    loaded = np.zeros(shape.num_experts, np.uint8)
    for t in range(2):
        r, ref, *_ = _run_and_check(shape, 13, xs[t], layer, ctx, pl, t, 2, cap, mode="host_master")
        # O10 on the hits / placement' just checked against the oracle chain
        io = oracle.io_step(r.hit_counts.cpu().numpy(), pl, r.placement.cpu().numpy(), loaded)
        assert r.stats["copies"] == io["copies"] and r.stats["promotions"] == io["promotions"]
        assert r.stats["h2d_bytes"] == r.stats["copies"] * shape.expert_bytes
        pl = r.placement.cpu().numpy()


# ------------------------------------------------------------------ ragged / edge cases
SMALL = g.Shape("small", 12, 3, 128, 192, 1, 40, steps=4, dtype="bf16", shared_expert=True)


@pytest.mark.parametrize("n", [1, 5, 17, 40])
def test_ragged_token_counts(n):
    layer = DeviceLayer(SMALL, 21)
    ctx = _ctx(SMALL, 12, max_tokens=40)
    x = g.block_hidden_np(SMALL, 21, steps=1, tokens=n)[0]
    _run_and_check(SMALL, 21, x, layer, ctx, np.zeros(12, np.uint8), 0, 1, 12)


def test_zero_tokens():
    from paper_2605_20179_b200 import tide
    layer = DeviceLayer(SMALL, 22)
    ctx = _ctx(SMALL, 12, max_tokens=40)
    x = torch.empty(0, SMALL.hidden, dtype=torch.bfloat16, device="cuda")
    r = ctx.moe_step(x, layer.router, **layer.weights(), placement=torch.zeros(12, dtype=torch.uint8, device="cuda"),
                     step=0, interval=1, stats=True)
    assert int(r.hit_counts.sum()) == 0 and r.stats["unique_experts"] == 0
    assert r.placement.cpu().numpy().tolist() == [1] * 12


def test_hot_expert_over_128_tokens():
    """An expert hit by > 128 tokens is split into several FFN work entries."""
    shape = g.Shape("hot", 4, 1, 128, 128, 1, 300, dtype="bf16")
    layer = DeviceLayer(shape, 23, skew=6.0)  # strong popularity bias -> one expert dominates
    ctx = _ctx(shape, 4)
    x = g.block_hidden_np(shape, 23, steps=1)[0]
    r, ref, *_ = _run_and_check(shape, 23, x, layer, ctx, np.zeros(4, np.uint8), 0, 1, 4)
    assert ref.hits.max() > 128


def test_k_equals_E_and_no_renorm():
    shape = g.Shape("kE", 8, 8, 64, 64, 1, 9, dtype="bf16")
    layer = DeviceLayer(shape, 24)
    ctx = _ctx(shape, 3, norm_topk=False)
    x = g.block_hidden_np(shape, 24, steps=1)[0]
    _run_and_check(shape, 24, x, layer, ctx, np.zeros(8, np.uint8), 0, 1, 3, norm_topk=False)


# ------------------------------------------------------------------ invariants (GPU-only)
def _out_bytes(ctx, layer, x, placement, step, interval, capacity, mode="device_all"):
    r = ctx.moe_step(x, layer.router, **layer.weights(mode),
                     placement=torch.from_numpy(placement).cuda(), step=step, interval=interval,
                     capacity=capacity)
    torch.cuda.synchronize()
    return r.out.view(torch.int16).cpu().numpy().copy()


def test_lossless_bitwise_across_placement_interval_capacity():
    """out is bitwise identical for any placement, interval and capacity,
    and between device_all (no offload) and host_master (pinned-host serving)."""
    from paper_2605_20179_b200 import tide
    shape = g.Shape("ll", 64, 8, 256, 256, 1, 32, dtype="bf16", shared_expert=True)
    layer = DeviceLayer(shape, 30, host_master=True)
    x = g.np_to_torch(g.block_hidden_np(shape, 30, steps=1)[0], "cuda")
    base = _out_bytes(tide.Context(desc_for(shape), 64), layer, x, np.zeros(64, np.uint8), 0, 1, 64)
    for cap, itv, step, mode in [(8, 1, 0, "device_all"), (8, 3, 1, "host_master"),
                                 (20, 2, 2, "host_master"), (64, 1, 0, "host_master"),
                                 (1, 5, 0, "host_master")]:
        ctx = tide.Context(desc_for(shape), cap, staging_slots=4)
        pl = g.random_placement(64, cap, cap + itv)
        got = _out_bytes(ctx, layer, x, pl, step, itv, cap, mode)
        assert (got == base).all(), (cap, itv, step, mode)


def test_repeat_runs_bitwise_identical():
    from paper_2605_20179_b200 import tide
    layer = DeviceLayer(g.MINI, 31)
    ctx = tide.Context(desc_for(g.MINI), 256)
    x = g.np_to_torch(g.block_hidden_np(g.MINI, 31, steps=1)[0], "cuda")
    a = _out_bytes(ctx, layer, x, np.zeros(256, np.uint8), 0, 1, 256)
    b = _out_bytes(ctx, layer, x, np.zeros(256, np.uint8), 0, 1, 256)
    assert (a == b).all()


def test_sweep_uniform_stress_parity_and_repeat():
    """Uniform iid routing at the sweep shape (256 tokens, ~all 256 experts hit, two shared
    entries): the FFN's phase-2 items wait on many entries' phase-1 counters and re-acquire
    their 32-entry windows often (ffn.cuh).  Every token against the oracle, and three
    repeats bitwise identical."""
    from paper_2605_20179_b200 import tide
    shape = g.SWEEP
    layer = DeviceLayer(shape, 13, skew=0.0)
    ctx = tide.Context(desc_for(shape), shape.num_experts)
    x_np = g.block_hidden_np(shape, 13, steps=1, iid=True)[0]
    r, ref, err, _ = _run_and_check(shape, 13, x_np, layer, ctx, np.zeros(256, np.uint8), 0, 1,
                                    shape.num_experts)
    assert int((r.hit_counts > 0).sum()) > 200
    x = g.np_to_torch(x_np, "cuda")
    outs = [_out_bytes(ctx, layer, x, np.zeros(256, np.uint8), 0, 1, 256) for _ in range(3)]
    assert all((o == outs[0]).all() for o in outs[1:])


def test_interval_one_and_io_model_match_oracle():
    """tau = 1 equals the per-step refresh policy, and the pinned-host I/O
    counters match the oracle's slot model (O10) step by step."""
    shape = g.Shape("io", 32, 4, 128, 128, 1, 16, steps=12, dtype="bf16")
    layer = DeviceLayer(shape, 32, host_master=True)
    for interval, lazy in [(1, False), (3, False), (4, True)]:
        ctx = _ctx(shape, 8, lazy=lazy, staging=4)
        xs = g.block_hidden_np(shape, 32)
        p = np.zeros(32, np.uint8)
        loaded = np.zeros(32, np.uint8)
        for t in range(shape.steps):
            r, ref, *_ = _run_and_check(shape, 32, xs[t], layer, ctx, p, t, interval, 8,
                                        mode="host_master")
            pl_new = r.placement.cpu().numpy()
            io = oracle.io_step(r.hit_counts.cpu().numpy(), p, pl_new, loaded, lazy=lazy)
            s = r.stats
            assert s["promotions"] == io["promotions"] and s["evictions"] == io["evictions"]
            assert s["experts_streamed"] == io["experts_streamed"], (t, s, io)
            assert s["copies"] == io["copies"], (t, s, io)
            assert s["resident_pairs"] == io["resident_pairs"]
            p = pl_new


def test_placement_over_capacity_rejected():
    from paper_2605_20179_b200 import tide
    layer = DeviceLayer(SMALL, 33, host_master=True)
    ctx = _ctx(SMALL, 4, max_tokens=40)
    x = g.np_to_torch(g.block_hidden_np(SMALL, 33, steps=1)[0], "cuda")
    with pytest.raises(tide.TideError) as ei:
        ctx.moe_step(x, layer.router, **layer.weights("host_master"),
                     placement=torch.ones(12, dtype=torch.uint8, device="cuda"), step=1,
                     interval=2)
    assert ei.value.status == tide.TIDE_EPLACEMENT


def test_invalid_arguments():
    from paper_2605_20179_b200 import tide
    layer = DeviceLayer(SMALL, 34)
    ctx = _ctx(SMALL, 4, max_tokens=40)
    x = g.np_to_torch(g.block_hidden_np(SMALL, 34, steps=1)[0], "cuda")
    pl = torch.zeros(12, dtype=torch.uint8, device="cuda")
    for kw, status in [(dict(interval=0), tide.TIDE_EINVAL), (dict(step=-1), tide.TIDE_EINVAL),
                       (dict(capacity=5), tide.TIDE_ECAPACITY)]:
        args = dict(placement=pl, step=0, interval=1)
        args.update(kw)
        with pytest.raises(tide.TideError) as ei:
            ctx.moe_step(x, layer.router, **layer.weights(), **args)
        assert ei.value.status == status
    with pytest.raises(tide.TideError):
        tide.Context(desc_for(SMALL), 13)
    with pytest.raises(tide.TideError):  # pageable host master
        ctx.moe_step(x, layer.router, host_master=layer.device_all.cpu(), shared_w=layer.shared,
                     placement=pl, step=0, interval=1)


def test_pack_expert_matches_concatenation():
    from paper_2605_20179_b200 import tide
    layer = DeviceLayer(SMALL, 35)
    n = layer.np
    d = desc_for(SMALL)
    dst = torch.empty(tide.expert_elems(d), dtype=torch.bfloat16, device="cuda")
    tide.pack_expert(d, g.np_to_torch(n.wg[3], "cuda"), g.np_to_torch(n.wu[3], "cuda"),
                     g.np_to_torch(n.wd[3]).pin_memory(), dst)
    torch.cuda.synchronize()
    assert torch.equal(dst, layer.device_all[3])
    assert tide.expert_bytes(d) == SMALL.expert_bytes


def test_device_generator_matches_host_bits():
    """tidegen's device twin produces the host generator's exact bytes."""
    wg, wu, wd = g.expert_torch(g.MINI, 7, 3, 17, "cuda")
    h = g.expert_np(g.MINI, 7, 3, 17)
    for a, b in zip((wg, wu, wd), h):
        assert (g.torch_to_np(a) == b).all()


@pytest.mark.parametrize("shape_name,tokens", [("mini", 32), ("mini", 256), ("flash", 32),
                                               ("flash", 200)])
def test_router_logit_error(shape_name, tokens):
    """R-17: the GPU's fp32 logits stay within 6e-7 of the fp64 oracle, so a routing flip
    needs an fp64 logit gap below ~1e-6 (which the near-tie flag covers)."""
    shape = g.SHAPES[shape_name]
    E, H = shape.num_experts, shape.hidden
    wr = g.router_np(shape, 51, 0)
    x = g.block_hidden_np(shape, 51, steps=1, tokens=tokens)[0]
    ref = oracle.router_logits(x, wr)
    sh = g.Shape(shape.name, E, shape.top_k, H, 64, 1, tokens, dtype="bf16")  # router only
    layer = DeviceLayer(sh, 51)
    from paper_2605_20179_b200 import tide
    ctx = tide.Context(desc_for(sh, max_tokens=tokens), E)
    r = ctx.moe_step(g.np_to_torch(x, "cuda"), g.np_to_torch(wr, "cuda"), **layer.weights(),
                     placement=torch.zeros(E, dtype=torch.uint8, device="cuda"), step=0,
                     interval=1, debug=True)
    torch.cuda.synchronize()
    err = np.abs(r.debug["logits"].cpu().numpy().astype(np.float64) - ref).max()
    assert err < 6e-7, f"max |logit - fp64| = {err:.3e}"


@pytest.mark.parametrize("E,H", [(1024, 128), (800, 256), (768, 256)])
def test_many_experts_work_list_paths(E, H):
    """E up to the descriptor limit: the FFN work list takes its batched path (E <= 768,
    at most 4 experts per thread) or its per-expert loop (E > 768); both against the oracle."""
    shape = g.Shape("wide", E, 4, H, 128, 1, 40, steps=1, dtype="bf16", shared_expert=True)
    layer = DeviceLayer(shape, 19)
    ctx = _ctx(shape, E)
    x = g.block_hidden_np(shape, 19, steps=1)[0]
    _run_and_check(shape, 19, x, layer, ctx, np.zeros(E, np.uint8), 0, 1, E)


def test_placement_over_capacity_device_all_leaves_placement_unchanged():
    """tide.h: on TIDE_EPLACEMENT (non-refresh step, popcount(placement) > C) placement_out is
    a copy of the input placement and hit_counts holds the step's hits (device_all mode
    reports the status when stats are requested)."""
    from paper_2605_20179_b200 import tide
    layer = DeviceLayer(SMALL, 36)
    ctx = _ctx(SMALL, 4, max_tokens=40)
    x_np = g.block_hidden_np(SMALL, 36, steps=1)[0]
    pin = torch.ones(12, dtype=torch.uint8, device="cuda")
    pout = torch.full((12,), 7, dtype=torch.uint8, device="cuda")
    hits = torch.full((12,), -1, dtype=torch.int32, device="cuda")
    with pytest.raises(tide.TideError) as ei:
        ctx.moe_step(g.np_to_torch(x_np, "cuda"), layer.router, **layer.weights(), placement=pin,
                     step=1, interval=2, placement_out=pout, hit_counts=hits, stats=True)
    assert ei.value.status == tide.TIDE_EPLACEMENT
    torch.cuda.synchronize()
    assert pout.cpu().numpy().tolist() == [1] * 12
    ref = oracle.moe_step(layer.oracle_layer(), x_np, SMALL.top_k, np.zeros(12, np.uint8), 0, 1, 12)
    assert (hits.cpu().numpy() == ref.hits).all()
