"""Small TIDE layer-steps for compute-sanitizer (memcheck / racecheck / synccheck).

usage: compute-sanitizer --tool <tool> --error-exitcode 9 python tools/sanitize_cases.py <case>
cases:
  toy_device_all    BJ.configs[0] shape (fp32 / tf32 MMA, CUDA-core router), every expert in HBM
  toy_host_master   the same with C = 4 < E: pinned-host serving, staged FFN chunks
  bf16_tc           bf16, tensor-core router (H split over 2 CTAs), shared expert
  graph_replay      bf16_tc captured in a CUDA graph per step and replayed
  p2p_world2        peer-memory expert parallelism, two ranks emulated in one process
Each case checks its outputs against the fp64 oracle (routing exact, output within 2e-2)
so a run is both a sanitizer pass and a parity pass.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import tidegen as g  # noqa: E402
from paper_2605_20179_b200 import tide  # noqa: E402
from tests._util import DeviceLayer, desc_for, rel_err, to_np_f64  # noqa: E402

BF = g.Shape("san", 32, 4, 512, 256, 1, 24, steps=4, dtype="bf16", shared_expert=True)


def check(shape, layer, x_np, r, placement, step, interval, cap):
    ref = oracle.moe_step(layer.oracle_layer(), x_np, shape.top_k, placement, step, interval, cap)
    assert ref.status == 0
    assert (r.hit_counts.cpu().numpy() == ref.hits).all(), "hits"
    assert (r.placement.cpu().numpy() == ref.placement).all(), "placement"
    err = rel_err(to_np_f64(r.out), ref.out)
    assert err < 2e-2, err
    return ref.placement


def run_steps(shape, mode, cap, steps=3, interval=2):
    layer = DeviceLayer(shape, 5, host_master=(mode == "host_master"))
    ctx = tide.Context(desc_for(shape), cap, 4)
    xs = g.block_hidden_np(shape, 5)
    p = np.zeros(shape.num_experts, np.uint8)
    for t in range(steps):
        r = ctx.moe_step(g.np_to_torch(xs[t], "cuda"), layer.router, **layer.weights(mode),
                         placement=torch.from_numpy(p).cuda(), step=t, interval=interval,
                         capacity=cap, stats=True)
        torch.cuda.synchronize()
        p = check(shape, layer, xs[t], r, p, t, interval, cap)
    print(f"{shape.name} {mode} C={cap}: {steps} steps ok")


def graph_replay():
    shape = BF
    E = shape.num_experts
    layer = DeviceLayer(shape, 6)
    ctx = tide.Context(desc_for(shape), E)
    xs = g.np_to_torch(g.block_hidden_np(shape, 6), "cuda")
    pl = torch.zeros(E, dtype=torch.uint8, device="cuda")
    out = torch.empty(shape.tokens, shape.hidden, dtype=torch.bfloat16, device="cuda")
    hits = torch.empty(E, dtype=torch.int32, device="cuda")
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        ctx.moe_step(xs[0], layer.router, **layer.weights(), placement=pl, step=0, interval=1,
                     out=out, hit_counts=hits, placement_out=pl)
    torch.cuda.current_stream().wait_stream(side)
    graphs = []
    for t in range(2):
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            ctx.moe_step(xs[t], layer.router, **layer.weights(), placement=pl, step=t,
                         interval=1, out=out, hit_counts=hits, placement_out=pl)
        graphs.append(gr)
    for t in range(2):
        graphs[t].replay()
        torch.cuda.synchronize()
        ref = oracle.moe_step(layer.oracle_layer(), g.torch_to_np(xs[t]), shape.top_k,
                              np.zeros(E, np.uint8), t, 1, E)
        assert (hits.cpu().numpy() == ref.hits).all()
        assert rel_err(to_np_f64(out), ref.out) < 2e-2
    print("graph replay: 2 captured steps ok")


def p2p_world2():
    shape = BF
    world, E = 2, BF.num_experts
    El = E // world
    layer = DeviceLayer(shape, 7)
    desc = desc_for(shape)
    warm = tide.EPPeerContext(desc, 0, 1)  # first use of every kernel before the two ranks run
    warm.connect(bases=[warm.export()[1]])
    warm.moe_step_ep(g.np_to_torch(g.block_hidden_np(shape, 7)[0], "cuda"), layer.router,
                     layer.device_all, shared_w=layer.shared,
                     placement=torch.zeros(E, dtype=torch.uint8, device="cuda"), step=0, interval=1)
    torch.cuda.synchronize()
    warm.close()
    ctxs = [tide.EPPeerContext(desc, r, world) for r in range(world)]
    bases = [c.export()[1] for c in ctxs]
    for c in ctxs:
        c.connect(bases=bases)
    streams = [torch.cuda.Stream() for _ in range(world)]
    local = [layer.device_all[r * El:(r + 1) * El].contiguous() for r in range(world)]
    xs = [g.block_hidden_np(shape, 70 + r) for r in range(world)]
    pl = [torch.zeros(El, dtype=torch.uint8, device="cuda") for _ in range(world)]
    outs = [torch.empty(shape.tokens, shape.hidden, dtype=torch.bfloat16, device="cuda")
            for _ in range(world)]
    hits = [torch.empty(E, dtype=torch.int32, device="cuda") for _ in range(world)]
    torch.cuda.synchronize()
    for t in range(2):
        xin = [g.np_to_torch(xs[r][t], "cuda") for r in range(world)]
        torch.cuda.synchronize()
        for r in range(world):
            with torch.cuda.stream(streams[r]):
                ctxs[r].moe_step_ep(xin[r], layer.router, local[r], shared_w=layer.shared,
                                    placement=pl[r], step=t, interval=1, out=outs[r],
                                    hit_counts=hits[r], placement_out=pl[r])
        torch.cuda.synchronize()
        x_cat = np.concatenate([xs[r][t] for r in range(world)])
        _, h, _, out = oracle.ep_step(layer.oracle_layer(), world, x_cat, shape.top_k,
                                      np.zeros(E, np.uint8), t, 1, El)
        for r in range(world):
            assert (hits[r].cpu().numpy() == h).all()
            n0 = r * shape.tokens
            assert rel_err(to_np_f64(outs[r]), out[n0:n0 + shape.tokens]) < 2e-2
    assert all(c.error() == 0 for c in ctxs)
    print("peer-memory EP, emulated world 2: 2 steps ok")


if __name__ == "__main__":
    case = sys.argv[1]
    torch.cuda.set_device(0)
    if case == "toy_device_all":
        run_steps(g.TOY, "device_all", g.TOY.num_experts)
    elif case == "toy_host_master":
        run_steps(g.TOY, "host_master", g.TOY.capacity, steps=4)
    elif case == "bf16_tc":
        run_steps(BF, "device_all", BF.num_experts)
    elif case == "graph_replay":
        graph_replay()
    elif case == "p2p_world2":
        p2p_world2()
    else:
        raise SystemExit(f"unknown case {case}")
