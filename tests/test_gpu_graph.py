"""NEXT-3 (CUDA graphs): tide_moe_step is stream-capturable in device_all mode.

The per-expert count buffers are double-buffered with a DEVICE parity word flipped by the
route kernel, so any captured sequence replays correctly, even when a context is called
an odd number of times per graph. Here each graph is one step t across the stack, so
every context is called once per graph. Two blocks are replayed from T per-step graphs and
compared bitwise with the eager stream: out, hit_counts, placement'. The eager outputs are
also checked against the oracle.
"""
import numpy as np
import pytest
import torch

import oracle
import tidegen as g
from tests._util import OUT_TOL, DeviceLayer, desc_for, rel_err, to_np_f64

pytestmark = pytest.mark.gpu

SHAPE = g.Shape("graph", 64, 8, 256, 256, 2, 24, steps=6, dtype="bf16", shared_expert=True)


def _stack(seed):
    from paper_2605_20179_b200 import tide
    desc = desc_for(SHAPE)
    E, N, H = SHAPE.num_experts, SHAPE.tokens, SHAPE.hidden
    out = []
    for l in range(SHAPE.layers):
        lay = DeviceLayer(SHAPE, seed, l)
        xs = g.block_hidden_np(SHAPE, seed, l)
        out.append(dict(lay=lay, ctx=tide.Context(desc, E),
                        x=torch.stack([g.np_to_torch(xs[t], "cuda") for t in range(SHAPE.steps)]),
                        xs=xs, pl=torch.zeros(E, dtype=torch.uint8, device="cuda"),
                        hits=torch.zeros(E, dtype=torch.int32, device="cuda"),
                        out=torch.zeros(N, H, dtype=torch.bfloat16, device="cuda")))
    return out


def _layer_step(L, t, interval):
    L["ctx"].moe_step(L["x"][t], L["lay"].router, **L["lay"].weights(), placement=L["pl"],
                      step=t, interval=interval, out=L["out"], hit_counts=L["hits"],
                      placement_out=L["pl"])


@pytest.mark.parametrize("interval", [1, 3])
def test_graph_replay_equals_eager(interval):
    T = SHAPE.steps
    eager, graphed = _stack(51), _stack(51)
    ref = []  # eager: two blocks
    for blk in range(2):
        for t in range(T):
            for L in eager:
                _layer_step(L, t, interval)
            ref.append([(L["out"].clone(), L["hits"].clone(), L["pl"].clone()) for L in eager])
    torch.cuda.synchronize()
    # oracle spot check of the eager stream (layer 0, block 0)
    L0 = eager[0]
    p = np.zeros(SHAPE.num_experts, np.uint8)
    for t in range(T):
        r = oracle.moe_step(L0["lay"].oracle_layer(), L0["xs"][t], SHAPE.top_k, p, t, interval,
                            SHAPE.num_experts)
        assert (ref[t][0][1].cpu().numpy() == r.hits).all()
        assert rel_err(to_np_f64(ref[t][0][0]), r.out) < OUT_TOL
        p = r.placement
    # capture one graph per step (warm up on a side stream first, as torch requires)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for L in graphed:
            _layer_step(L, 0, interval)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    for L in graphed:
        L["pl"].zero_()
    graphs = []
    for t in range(T):
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            for L in graphed:
                _layer_step(L, t, interval)
        graphs.append(gr)
    torch.cuda.synchronize()
    # capture ran nothing: reset placement state and replay two blocks
    for L in graphed:
        L["pl"].zero_()
    i = 0
    for blk in range(2):
        for t in range(T):
            graphs[t].replay()
            for L, (o, h, pl) in zip(graphed, ref[i]):
                torch.cuda.synchronize()
                assert torch.equal(L["hits"], h), (blk, t)
                assert torch.equal(L["pl"], pl), (blk, t)
                assert torch.equal(L["out"].view(torch.int16), o.view(torch.int16)), (blk, t)
            i += 1


def test_cross_layer_prefetch_is_bitwise_neutral():
    """NEXT-3 prefetch (tide_ctx_set_prefetch, ring over the stack) is a cache hint: every
    output, hit count and placement equals the run without it, bit for bit."""
    from paper_2605_20179_b200 import tide
    T = SHAPE.steps
    plain, pf = _stack(53), _stack(53)
    n = len(pf)
    for i, L in enumerate(pf):
        nx = pf[(i + 1) % n]
        L["ctx"].set_prefetch(nx["ctx"], nx["lay"].device_all, 1 << 30)
    for t in range(T):
        for A, B in zip(plain, pf):
            _layer_step(A, t, 2)
            _layer_step(B, t, 2)
            torch.cuda.synchronize()
            assert torch.equal(A["out"].view(torch.int16), B["out"].view(torch.int16)), t
            assert torch.equal(A["hits"], B["hits"]) and torch.equal(A["pl"], B["pl"])
    with pytest.raises(tide.TideError):
        pf[0]["ctx"].set_prefetch(pf[1]["ctx"], pf[1]["lay"].device_all, -1)
    pf[0]["ctx"].set_prefetch(None)  # disable
