"""Peer-memory expert parallelism (tide_ctx_create_ep_p2p): the EP step with dispatch and
combine done by the kernels over peer memory instead of NCCL (include/tide.h, ep.cuh).

- world = 1: bitwise equal to the NCCL EP path and to the single-device step.
- world = 2 and 4, emulated on ONE B200 inside one process: one context per rank, each
  stepping on its own CUDA stream, peers addressed through plain device pointers
  (tide_ctx_ep_connect with `bases`).  The kernels run the real protocol (stores into
  the peers' symmetric regions, release/acquire counters at system scope, parity
  double-buffering); checked against the oracle's EP emulation (O11):
  global hits and per-rank placements exact, outputs within the north-star tolerance,
  and bitwise equal to the single-device step on all ranks' tokens, over several steps
  with ragged per-rank token counts; bitwise repeatable.
- world = 2 across two PROCESSES on one B200, peers mapped with CUDA IPC
  (tide_ctx_ep_export / connect with `handles`), the multi-process setup path.
"""
import os
import socket

import numpy as np
import pytest
import torch

import oracle
import tidegen as g
from tests._util import OUT_TOL, DeviceLayer, desc_for, rel_err, to_np_f64

pytestmark = pytest.mark.gpu

SHAPE = g.Shape("ep", 32, 4, 256, 256, 1, 24, steps=4, dtype="bf16", shared_expert=True)


def test_p2p_world1_equals_nccl_and_single_device():
    from paper_2605_20179_b200 import tide
    layer = DeviceLayer(SHAPE, 51)
    desc = desc_for(SHAPE)
    p2p = tide.EPPeerContext(desc, 0, 1)
    nccl = tide.EPContext(desc, tide.nccl_unique_id(), 0, 1)
    single = tide.Context(desc, SHAPE.num_experts)
    E = SHAPE.num_experts
    xs = g.block_hidden_np(SHAPE, 51)
    pl = [torch.zeros(E, dtype=torch.uint8, device="cuda") for _ in range(3)]
    for t in range(SHAPE.steps):
        for n in (SHAPE.tokens, 7):  # full and ragged blocks
            x = g.np_to_torch(xs[t][:n], "cuda")
            a = p2p.moe_step_ep(x, layer.router, layer.device_all, shared_w=layer.shared,
                                placement=pl[0], step=t, interval=2)
            b = nccl.moe_step_ep(x, layer.router, layer.device_all, shared_w=layer.shared,
                                 placement=pl[1], step=t, interval=2)
            c = single.moe_step(x, layer.router, **layer.weights(), placement=pl[2], step=t,
                                interval=2)
            torch.cuda.synchronize()
            for r in (b, c):
                assert torch.equal(a.out.view(torch.int16), r.out.view(torch.int16)), (t, n)
                assert torch.equal(a.hit_counts, r.hit_counts)
                assert torch.equal(a.placement, r.placement)
            for p, r in zip(pl, (a, b, c)):
                p.copy_(r.placement)
    assert p2p.error() == 0


def _emulated(world, seed, tokens, steps, interval, cap_r):
    """Run `steps` EP steps of `world` emulated ranks; returns per-step per-rank results."""
    from paper_2605_20179_b200 import tide
    layer = DeviceLayer(SHAPE, seed)
    desc = desc_for(SHAPE)
    E = SHAPE.num_experts
    El = E // world
    # one-process emulation only: a first step of this shape on a world-1 context, so no
    # first-use host work (module loading, allocator growth) can stall the host between
    # two emulated ranks' enqueues while the first rank's kernels wait for the second
    warm = tide.EPPeerContext(desc, 0, 1)
    warm.connect(bases=[warm.export()[1]])
    warm.moe_step_ep(g.np_to_torch(g.block_hidden_np(SHAPE, seed)[0], "cuda"), layer.router,
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
    xs = [g.block_hidden_np(SHAPE, seed + 100 * (r + 1)) for r in range(world)]
    pl = [torch.zeros(El, dtype=torch.uint8, device="cuda") for _ in range(world)]
    torch.cuda.synchronize()
    res = []
    # every buffer exists before any rank is enqueued: a device allocation between two
    # ranks' enqueues would synchronise the device while the first rank waits for the second
    outs_buf = [torch.empty(tokens[r], SHAPE.hidden, dtype=torch.bfloat16, device="cuda")
                for r in range(world)]
    hits_buf = [torch.empty(E, dtype=torch.int32, device="cuda") for _ in range(world)]
    for t in range(steps):
        xin = [g.np_to_torch(xs[r][t % SHAPE.steps][:tokens[r]], "cuda") for r in range(world)]
        torch.cuda.synchronize()
        outs = []
        for r in range(world):  # enqueue every rank; the kernels synchronise each other
            with torch.cuda.stream(streams[r]):
                outs.append(ctxs[r].moe_step_ep(xin[r], layer.router, local[r],
                                                shared_w=layer.shared, placement=pl[r], step=t,
                                                interval=interval, capacity=cap_r,
                                                out=outs_buf[r], hit_counts=hits_buf[r],
                                                placement_out=pl[r]))
        torch.cuda.synchronize()
        res.append([(to_np_f64(o.out), o.hit_counts.cpu().numpy(), o.placement.cpu().numpy(),
                     o.out.view(torch.int16).cpu().numpy()) for o in outs])
    for c in ctxs:
        assert c.error() == 0, "peer-memory wait timed out"
    return layer, xs, res


@pytest.mark.parametrize("world,tokens,cap_r", [(2, (24, 17), 10), (4, (24, 5, 0, 13), 3)])
def test_p2p_emulated_world_matches_oracle_ep(world, tokens, cap_r):
    """Per rank: hits and placement' exact vs the oracle's EP emulation (O11), outputs within
    2e-2 of it, and every output bit equal to the single-device step on all ranks' tokens
    (the combine runs the single-device arithmetic on the pairs' y rows)."""
    from paper_2605_20179_b200 import tide
    steps, interval = 4, 2
    layer, xs, res = _emulated(world, 61, tokens, steps, interval, cap_r)
    E, k = SHAPE.num_experts, SHAPE.top_k
    El = E // world
    ol = layer.oracle_layer()
    p_in = np.zeros(E, np.uint8)
    single = tide.Context(desc_for(SHAPE, max_tokens=sum(tokens)), E)
    p1 = torch.zeros(E, dtype=torch.uint8, device="cuda")
    for t in range(steps):
        x_cat = np.concatenate([xs[r][t % SHAPE.steps][:tokens[r]] for r in range(world)])
        _, hits, pout, out = oracle.ep_step(ol, world, x_cat, k, p_in, t, interval, cap_r)
        one = single.moe_step(g.np_to_torch(x_cat, "cuda"), layer.router, **layer.weights(),
                              placement=p1, step=t, interval=interval, placement_out=p1)
        torch.cuda.synchronize()
        one_out = one.out.view(torch.int16).cpu().numpy()
        row = 0
        for r in range(world):
            o, h, p, _ = res[t][r]
            assert (h == hits).all(), (t, r)
            assert (p == pout[r * El:(r + 1) * El]).all(), (t, r)
            if tokens[r]:
                err = rel_err(o, out[row:row + tokens[r]])
                assert err < OUT_TOL, (t, r, err)
                ob = res[t][r][3]
                assert np.array_equal(ob, one_out[row:row + tokens[r]]), (t, r)
            row += tokens[r]
        p_in = pout


def test_p2p_emulated_repeat_bitwise():
    _, _, a = _emulated(2, 71, (24, 24), 3, 1, 16)
    _, _, b = _emulated(2, 71, (24, 24), 3, 1, 16)
    for ra, rb in zip(a, b):
        for (oa, ha, pa, _), (ob, hb, pb, _) in zip(ra, rb):
            assert np.array_equal(oa, ob) and np.array_equal(ha, hb) and np.array_equal(pa, pb)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _ipc_rank(rank, world, port, q):
    import torch.distributed as dist
    from paper_2605_20179_b200 import tide
    try:
        torch.cuda.set_device(0)  # both processes on the one GPU: IPC-mapped peer regions
        os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        layer = DeviceLayer(SHAPE, 81)
        desc = desc_for(SHAPE)
        E, k = SHAPE.num_experts, SHAPE.top_k
        El = E // world
        ctx = tide.EPPeerContext(desc, rank, world)
        handles = [None] * world
        dist.all_gather_object(handles, ctx.export()[0])
        ctx.connect(handles=handles)
        dist.barrier()
        xs = [g.block_hidden_np(SHAPE, 900 + r, steps=2) for r in range(world)]
        pl = torch.zeros(El, dtype=torch.uint8, device="cuda")
        p_in = np.zeros(E, np.uint8)
        errs, ok = [], True
        for t in range(2):
            r = ctx.moe_step_ep(g.np_to_torch(xs[rank][t], "cuda"), layer.router,
                                layer.device_all[rank * El:(rank + 1) * El].contiguous(),
                                shared_w=layer.shared, placement=pl, step=t, interval=1,
                                capacity=El // 2, placement_out=pl)
            torch.cuda.synchronize()
            x_cat = np.concatenate([xs[i][t] for i in range(world)])
            _, hits, pout, out = oracle.ep_step(layer.oracle_layer(), world, x_cat, k, p_in, t, 1,
                                                El // 2)
            n = SHAPE.tokens
            errs.append(rel_err(to_np_f64(r.out), out[rank * n:(rank + 1) * n]))
            ok &= bool((r.hit_counts.cpu().numpy() == hits).all())
            ok &= bool((r.placement.cpu().numpy() == pout[rank * El:(rank + 1) * El]).all())
            p_in = pout
        ok &= ctx.error() == 0
        dist.barrier()  # every rank done before any region is unmapped / freed
        ctx.close()
        q.put((rank, max(errs), ok))
        dist.destroy_process_group()
    except Exception as ex:
        q.put((rank, repr(ex), False))


def test_p2p_two_processes_ipc():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    for rank, err, ok in res:
        assert not isinstance(err, str), err
        assert ok and err < OUT_TOL, (rank, err)


def test_p2p_emulated_world2_mini_shape_bitwise():
    """BJ.configs[1] layer shape (E=256 top-8 + shared expert, H=2048, F=512), two emulated
    ranks with a block of 32 tokens each, 3 steps: every output bit, the global hits and each
    rank's placement equal the single-device step on the 64 tokens."""
    from paper_2605_20179_b200 import tide
    s = g.MINI
    world, N, E = 2, s.tokens, s.num_experts
    El = E // world
    layer = DeviceLayer(s, 91)
    desc = desc_for(s)
    warm = tide.EPPeerContext(desc, 0, 1)
    warm.connect(bases=[warm.export()[1]])
    warm.moe_step_ep(g.np_to_torch(g.block_hidden_np(s, 91, steps=1)[0], "cuda"), layer.router,
                     layer.device_all, shared_w=layer.shared,
                     placement=torch.zeros(E, dtype=torch.uint8, device="cuda"), step=0, interval=1)
    torch.cuda.synchronize()
    warm.close()
    ctxs = [tide.EPPeerContext(desc, r, world) for r in range(world)]
    bases = [c.export()[1] for c in ctxs]
    for c in ctxs:
        c.connect(bases=bases)
    single = tide.Context(desc_for(s, max_tokens=world * N), E)
    streams = [torch.cuda.Stream() for _ in range(world)]
    local = [layer.device_all[r * El:(r + 1) * El].contiguous() for r in range(world)]
    xs = [g.block_hidden_np(s, 500 + r, steps=3) for r in range(world)]
    pl = [torch.zeros(El, dtype=torch.uint8, device="cuda") for _ in range(world)]
    p1 = torch.zeros(E, dtype=torch.uint8, device="cuda")
    outs = [torch.empty(N, s.hidden, dtype=torch.bfloat16, device="cuda") for _ in range(world)]
    hits = [torch.empty(E, dtype=torch.int32, device="cuda") for _ in range(world)]
    for t in range(3):
        xin = [g.np_to_torch(xs[r][t], "cuda") for r in range(world)]
        torch.cuda.synchronize()
        for r in range(world):
            with torch.cuda.stream(streams[r]):
                ctxs[r].moe_step_ep(xin[r], layer.router, local[r], shared_w=layer.shared,
                                    placement=pl[r], step=t, interval=2, capacity=El // 2,
                                    out=outs[r], hit_counts=hits[r], placement_out=pl[r])
        torch.cuda.synchronize()
        one = single.moe_step(torch.cat(xin), layer.router, **layer.weights(), placement=p1,
                              step=t, interval=2, placement_out=p1)
        torch.cuda.synchronize()
        for r in range(world):
            assert torch.equal(outs[r].view(torch.int16), one.out[r * N:(r + 1) * N].view(torch.int16)), (t, r)
            assert torch.equal(hits[r], one.hit_counts), (t, r)
    for c in ctxs:
        assert c.error() == 0


def test_p2p_emulated_world2_toy_fp32():
    """BJ.configs[0] shapes (fp32, tf32 MMA, CUDA-core router): two emulated ranks, the peer
    path's fp32 instances; bitwise equal to the single-device step, hits exact."""
    from paper_2605_20179_b200 import tide
    s = g.TOY
    world, N, E = 2, s.tokens, s.num_experts
    El = E // world
    layer = DeviceLayer(s, 95)
    desc = desc_for(s)
    warm = tide.EPPeerContext(desc, 0, 1)
    warm.connect(bases=[warm.export()[1]])
    warm.moe_step_ep(g.np_to_torch(g.block_hidden_np(s, 95, steps=1)[0], "cuda"), layer.router,
                     layer.device_all, placement=torch.zeros(E, dtype=torch.uint8, device="cuda"),
                     step=0, interval=1)
    torch.cuda.synchronize()
    warm.close()
    ctxs = [tide.EPPeerContext(desc, r, world) for r in range(world)]
    bases = [c.export()[1] for c in ctxs]
    for c in ctxs:
        c.connect(bases=bases)
    single = tide.Context(desc_for(s, max_tokens=world * N), E)
    streams = [torch.cuda.Stream() for _ in range(world)]
    local = [layer.device_all[r * El:(r + 1) * El].contiguous() for r in range(world)]
    xs = [g.block_hidden_np(s, 700 + r, steps=4) for r in range(world)]
    pl = [torch.zeros(El, dtype=torch.uint8, device="cuda") for _ in range(world)]
    p1 = torch.zeros(E, dtype=torch.uint8, device="cuda")
    outs = [torch.empty(N, s.hidden, dtype=torch.float32, device="cuda") for _ in range(world)]
    hits = [torch.empty(E, dtype=torch.int32, device="cuda") for _ in range(world)]
    for t in range(4):
        xin = [g.np_to_torch(xs[r][t], "cuda") for r in range(world)]
        torch.cuda.synchronize()
        for r in range(world):
            with torch.cuda.stream(streams[r]):
                ctxs[r].moe_step_ep(xin[r], layer.router, local[r], placement=pl[r], step=t,
                                    interval=s.interval, capacity=s.capacity // world,
                                    out=outs[r], hit_counts=hits[r], placement_out=pl[r])
        torch.cuda.synchronize()
        one = single.moe_step(torch.cat(xin), layer.router, **layer.weights(), placement=p1,
                              step=t, interval=s.interval, placement_out=p1)
        torch.cuda.synchronize()
        for r in range(world):
            assert torch.equal(outs[r].view(torch.int32), one.out[r * N:(r + 1) * N].view(torch.int32)), (t, r)
            assert torch.equal(hits[r], one.hit_counts), (t, r)
    for c in ctxs:
        assert c.error() == 0


def test_p2p_world1_graph_replay_bitwise():
    """The peer-memory EP step holds no host state per call (parity-double-buffered counters):
    per-step CUDA graphs of it replay bitwise equal to the single-device step, over two blocks."""
    from paper_2605_20179_b200 import tide
    layer = DeviceLayer(SHAPE, 97)
    desc = desc_for(SHAPE)
    E, N, T = SHAPE.num_experts, SHAPE.tokens, SHAPE.steps
    ctx = tide.EPPeerContext(desc, 0, 1)
    ctx.connect(bases=[ctx.export()[1]])
    single = tide.Context(desc, E)
    xs = torch.stack([g.np_to_torch(x, "cuda") for x in g.block_hidden_np(SHAPE, 97)])
    pl, p1 = (torch.zeros(E, dtype=torch.uint8, device="cuda") for _ in range(2))
    out = torch.empty(N, SHAPE.hidden, dtype=torch.bfloat16, device="cuda")
    hits = torch.empty(E, dtype=torch.int32, device="cuda")

    def step(t):
        ctx.moe_step_ep(xs[t], layer.router, layer.device_all, shared_w=layer.shared,
                        placement=pl, step=t, interval=2, out=out, hit_counts=hits,
                        placement_out=pl)

    s = torch.cuda.Stream()  # warm-up off the capture stream, as torch requires
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step(0)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    graphs = []
    for t in range(T):
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            step(t)
        graphs.append(gr)
    torch.cuda.synchronize()
    pl.zero_()
    for blk in range(2):
        for t in range(T):
            graphs[t].replay()
            ref = single.moe_step(xs[t], layer.router, **layer.weights(), placement=p1, step=t,
                                  interval=2, placement_out=p1)
            torch.cuda.synchronize()
            assert torch.equal(out.view(torch.int16), ref.out.view(torch.int16)), (blk, t)
            assert torch.equal(hits, ref.hit_counts) and torch.equal(pl, p1), (blk, t)
    assert ctx.error() == 0
