"""Parity at BASELINE.json's full size in the launch configuration bench.py times.

BJ.configs[1]: the 20-layer LLaDA2.0-mini-shaped stack (E=256 top-8 + shared expert,
H=2048, F=512), a block of 32 tokens, C = E, refresh interval 4, weights generated on the
device and packed by tide_pack_expert, the NEXT-3 cross-layer L2 prefetch ring (32 MB), one
CUDA graph per block step t holding every layer-step of the stack, replayed for a whole
block (T = 32 steps).  Each captured layer-step also copies its routing outputs (top-k,
gates, pos, order, offsets) into per-(layer, step) buffers (tide.py debug="routing"), so
against the fp64 oracle on the same bytes:

* every layer at every step: top-k of every token bit-exact (near-tie tokens, R-17, accept
  either selection), and hits, placement', order, offsets and pos bit-exact against the
  oracle's O4-O7 fed the GPU's routing on flagged steps (the routing the placement chain
  actually saw), gates within 1e-4;
* outputs of every token within 2e-2 at every layer of the steps in FULL_STEPS (refresh and
  skipped steps, early and late in the block) and at the layers in EVERY_STEP_LAYERS for
  every step of the block.
"""
import numpy as np
import pytest
import torch

import oracle
import tidegen as g
from tests._util import OUT_TOL, check_routing, rel_err, to_np_f64

pytestmark = pytest.mark.gpu

INTERVAL = 4
FULL_STEPS = (0, 1, 2, 5, 16, 31)   # every token, every layer
EVERY_STEP_LAYERS = (0, 9, 19)      # every token, every step


def test_mini_stack_graphs_prefetch_full_block():
    from paper_2605_20179_b200 import tide
    s, seed, dev = g.MINI, 7, torch.device("cuda", 0)
    E, k, H, F, N, T = s.num_experts, s.top_k, s.hidden, s.ffn, s.tokens, s.steps
    desc = tide.make_desc(E, k, H, F, N, tide.TIDE_BF16, shared_expert=True)
    layers, host = [], []
    to = g.torch_to_np
    for l in range(s.layers):
        wr, wg, wu, wd, sh = g.layer_torch(s, seed, l, dev)
        host.append(oracle.Layer(to(wr), to(wg), to(wu), to(wd), tuple(to(a) for a in sh)))
        packed = tide.pack_layer(desc, wg, wu, wd)
        del wg, wu, wd
        layers.append(dict(router=wr, w=packed, shared=torch.cat([a.reshape(-1) for a in sh]),
                           ctx=tide.Context(desc, E, 16, 0),
                           x=g.block_hidden_torch(s, seed, l, dev),
                           pl=torch.zeros(E, dtype=torch.uint8, device=dev),
                           hits=torch.empty(T, E, dtype=torch.int32, device=dev),
                           plo=torch.empty(T, E, dtype=torch.uint8, device=dev),
                           out=torch.empty(T, N, H, dtype=torch.bfloat16, device=dev),
                           dbg=[None] * T))
    torch.cuda.empty_cache()
    for li, L in enumerate(layers):  # prefetch ring, as bench.py
        nx = layers[(li + 1) % len(layers)]
        L["ctx"].set_prefetch(nx["ctx"], nx["w"], 32_000_000)

    def step(L, t, debug=False):
        r = L["ctx"].moe_step(L["x"][t], L["router"], device_all=L["w"], shared_w=L["shared"],
                              placement=L["pl"], step=t, interval=INTERVAL, out=L["out"][t],
                              hit_counts=L["hits"][t], placement_out=L["pl"],
                              debug="routing" if debug else False)
        if debug:
            L["dbg"][t] = r.debug  # buffers from the graph's pool, written at every replay

    # warm up on a side stream (torch graph-capture requirement), then capture per-step graphs
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for L in layers:
            step(L, 0)
    torch.cuda.current_stream().wait_stream(side)
    graphs = []
    for t in range(T):
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            for L in layers:
                step(L, t, debug=True)
                L["plo"][t].copy_(L["pl"])  # placement' of (layer, t), kept for the check
        graphs.append(gr)
    torch.cuda.synchronize()
    for L in layers:
        L["pl"].zero_()
    for t in range(T):
        graphs[t].replay()
    torch.cuda.synchronize()

    worst, n_flagged, n_out = 0.0, 0, 0
    for l, L in enumerate(layers):
        p_prev = np.zeros(E, np.uint8)
        xs = to(L["x"])
        hits_all, plo_all, out_all = (L["hits"].cpu().numpy(), L["plo"].cpu().numpy(),
                                      to_np_f64(L["out"]))
        for t in range(T):
            d = {kk: v.cpu().numpy() for kk, v in L["dbg"][t].items() if v is not None}
            logits = oracle.router_logits(xs[t], host[l].wr)
            ref_topk = oracle.topk(logits, k)
            flagged = check_routing(d["topk_idx"], logits, ref_topk, k)
            n_flagged += int(flagged.sum())
            topk = d["topk_idx"] if flagged.any() else ref_topk
            hits = oracle.hits(topk, E)
            pl_ref = oracle.placement(hits, E, oracle.is_refresh(t, INTERVAL), p_prev)
            order, offsets, pos = oracle.buckets(topk, pl_ref)
            assert (hits_all[t] == hits).all(), (l, t)
            assert (plo_all[t] == pl_ref).all(), (l, t)
            assert (d["order"] == order).all() and (d["offsets"] == offsets).all(), (l, t)
            assert (d["pos"] == pos).all(), (l, t)
            gates = oracle.gates(logits, topk, True)
            assert np.abs(d["gates"] - gates).max() < 1e-4, (l, t)
            p_prev = pl_ref
            if t in FULL_STEPS or l in EVERY_STEP_LAYERS:
                ref_out = oracle.combine(host[l], xs[t], topk, gates)
                err = rel_err(out_all[t], ref_out)
                assert err < OUT_TOL, (l, t, err)
                worst = max(worst, err)
                n_out += 1
    print(f"full-size mini stack, graphs + prefetch, T={T}: routing/hits/placement/pos exact at "
          f"{len(layers)} layers x {T} steps ({n_flagged} near-tie tokens flagged); every "
          f"token's output at {n_out} layer-steps, worst rel err {worst:.3e}")
