"""Exact logit ties through the GPU router: the lowest expert id wins (DESIGN R-3).

Routers are built so that several experts have *bitwise identical* logits on both sides
(identical router rows, or an all-zero router), so these tokens are not near-tie flagged
(tests/_util.near_tie_tokens flags only 0 < gap < 1e-6): the selection and its order must
equal the oracle's lowest-id rule exactly, and every downstream stage (hits, placement,
buckets, pos, gates, output) is checked against the oracle as in the parity tests.

Tie positions are chosen to exercise every comparison the top-k makes (route.cuh
route_token): two tied experts in the same lane's register list (e and e + 32), tied
experts in different lanes (warp argmax on redux.sync), tied experts in different MMA
tiles and different halves of a tile (router phase 1), and a tie across the k / k+1
selection boundary.
"""
import numpy as np
import pytest
import torch

import oracle
import tidegen as g
from tests._util import DeviceLayer, OUT_TOL, desc_for, near_tie_tokens, rel_err, to_np_f64

pytestmark = pytest.mark.gpu


def _set_router(layer: DeviceLayer, wr_bits: np.ndarray):
    layer.np.wr = wr_bits
    layer.router = g.np_to_torch(wr_bits, "cuda")


def _step(shape, layer, x_np, capacity=None, step=0, interval=1):
    from paper_2605_20179_b200 import tide
    E, k = shape.num_experts, shape.top_k
    cap = capacity or E
    ctx = tide.Context(desc_for(shape), cap)
    pl = np.zeros(E, np.uint8)
    r = ctx.moe_step(g.np_to_torch(x_np, "cuda"), layer.router, **layer.weights(),
                     placement=torch.from_numpy(pl).cuda(), step=step, interval=interval,
                     capacity=cap, stats=True, debug=True)
    torch.cuda.synchronize()
    ref = oracle.moe_step(layer.oracle_layer(), x_np, k, pl, step, interval, cap)
    assert ref.status == 0
    gt = r.debug["topk_idx"].cpu().numpy()
    assert not near_tie_tokens(ref.logits, k).any(), "construction left a non-exact near tie"
    assert (gt == ref.topk_idx).all(), (gt[:4], ref.topk_idx[:4])  # strict: no flagging
    assert (r.hit_counts.cpu().numpy() == ref.hits).all()
    assert (r.placement.cpu().numpy() == ref.placement).all()
    assert (r.debug["order"].cpu().numpy() == ref.order).all()
    assert (r.debug["offsets"].cpu().numpy() == ref.offsets).all()
    assert (r.debug["pos"].cpu().numpy() == ref.pos).all()
    assert np.abs(r.debug["gates"].cpu().numpy() - ref.gates).max() < 1e-4
    err = rel_err(to_np_f64(r.out), ref.out)
    assert err < OUT_TOL, err
    return gt, ref, r


def _bits(shape, a32):
    return g.f32_to_bf16_bits(a32.astype(np.float32)) if shape.dtype == "bf16" else a32.astype(np.float32)


def _f32(shape, bits):
    return g.bf16_bits_to_f32(bits) if shape.dtype == "bf16" else bits.astype(np.float32)


TC = g.Shape("tie_tc", 256, 8, 256, 128, 1, 24, dtype="bf16", shared_expert=True)   # tensor-core router
CC = g.Shape("tie_cc", 48, 4, 128, 128, 1, 20, dtype="bf16")                         # CUDA-core router (E % 16 != 0 path not taken: H % 256 != 0)
F32 = g.Shape("tie_f32", 16, 2, 64, 128, 1, 8, dtype="f32")                           # fp32 router (toy kind)


@pytest.mark.parametrize("shape", [TC, CC, F32], ids=lambda s: s.name)
def test_zero_router_selects_lowest_ids(shape):
    """Wr = 0: every logit is exactly 0, so every token selects experts 0..k-1 in id order
    with gates 1/k (O1 pin's GPU counterpart)."""
    layer = DeviceLayer(shape, 61)
    _set_router(layer, _bits(shape, np.zeros((shape.num_experts, shape.hidden), np.float32)))
    x = g.block_hidden_np(shape, 61, steps=1)[0]
    gt, ref, r = _step(shape, layer, x)
    want = np.tile(np.arange(shape.top_k, dtype=np.int32), (shape.tokens, 1))
    assert (gt == want).all()
    assert np.allclose(r.debug["gates"].cpu().numpy(), 1.0 / shape.top_k, atol=1e-6)
    assert (r.hit_counts.cpu().numpy()[: shape.top_k] == shape.tokens).all()


def _dominant_tied(shape, seed, tied, bias):
    """Router whose rows `tied` are one shared random row with bias `bias` in column 0 (the
    x[:, 0] == 1 column), so those experts have identical logits that exceed all others."""
    E, H = shape.num_experts, shape.hidden
    w = _f32(shape, g.router_np(shape, seed, 0, skew=0.0)).astype(np.float32).copy()
    row = w[tied[0]].copy()
    row[0] = bias
    for e in tied:
        w[e] = row
    return _bits(shape, w)


@pytest.mark.parametrize("shape,tied", [
    (TC, [200, 140, 35, 3]),  # lanes 8/12/3/3, register slots 6/4/1/0, MMA tiles 12/8/2/0
    (CC, [47, 32, 16, 0]),  # 0 and 32 share lane 0 (register slots 0 and 1)
    (F32, [14, 9, 5]),
], ids=["tc", "cc", "f32"])
def test_duplicated_rows_rank_by_id(shape, tied):
    """Experts with identical router rows tie exactly; they occupy the top slots in
    ascending id order whatever their lane, register slot or MMA tile."""
    layer = DeviceLayer(shape, 62)
    _set_router(layer, _dominant_tied(shape, 62, tied, 20.0))
    x = g.block_hidden_np(shape, 62, steps=1)[0]
    gt, ref, r = _step(shape, layer, x)
    want = sorted(tied)[: shape.top_k]
    assert (gt[:, : len(want)] == np.array(want, np.int32)).all(), gt[:3]
    gates = r.debug["gates"].cpu().numpy()
    assert np.allclose(gates[:, : len(want)], gates[:, :1], rtol=0, atol=0)  # tied -> equal gates


@pytest.mark.parametrize("shape", [TC, CC], ids=lambda s: s.name)
def test_tie_across_the_k_boundary(shape):
    """k-1 dominant experts with distinct logits, then three experts tied for the k-th slot:
    only the lowest id of the three is selected, the other two are not."""
    E, H, k = shape.num_experts, shape.hidden, shape.top_k
    rng = np.random.default_rng(63)
    ids = rng.permutation(E)
    dom, trio = ids[: k - 1], ids[k - 1: k + 2]
    w = _f32(shape, g.router_np(shape, 63, 0, skew=0.0)).astype(np.float32).copy()
    base = w[dom[0]].copy()
    for i, e in enumerate(dom):  # identical rows but column 0: logits exactly 1.0 apart
        w[e] = base
        w[e, 0] = 40.0 - i
    for e in trio:
        w[e] = base
        w[e, 0] = 40.0 - k - 1.0
    layer = DeviceLayer(shape, 63)
    _set_router(layer, _bits(shape, w))
    x = g.block_hidden_np(shape, 63, steps=1)[0]
    gt, ref, r = _step(shape, layer, x, capacity=max(1, E // 4))
    assert (gt[:, : k - 1] == dom.astype(np.int32)).all()
    assert (gt[:, k - 1] == int(trio.min())).all()
    others = set(int(e) for e in trio) - {int(trio.min())}
    assert not np.isin(gt, list(others)).any()


def test_placement_ties_lowest_id_at_refresh():
    """Hit-count ties at the capacity boundary (a4, R-8): with every token routed to the same
    tied experts, placement' keeps the lowest ids among equal counts."""
    shape = TC
    tied = [250, 130, 64, 1]
    layer = DeviceLayer(shape, 64)
    _set_router(layer, _dominant_tied(shape, 64, tied, 20.0))
    x = g.block_hidden_np(shape, 64, steps=1)[0]
    gt, ref, r = _step(shape, layer, x, capacity=2)
    pl = r.placement.cpu().numpy()
    hits = r.hit_counts.cpu().numpy()
    assert (hits[tied] == shape.tokens).all()
    top = np.nonzero(hits == hits.max())[0]  # >= 4 experts share the maximum count
    assert sorted(np.nonzero(pl)[0].tolist()) == sorted(top.tolist())[:2]
