"""Expert-parallel step (tide_moe_step_ep) through the C ABI and NCCL.

world = 1 runs on any single B200 (the full code path: NCCL all-gather dispatch, local
grouped FFN, partial sums, NCCL all-to-all, rank-order sum); it must equal the
single-device step bitwise and the oracle within tolerance.  world = 2 needs two GPUs
(one process per GPU) and is skipped otherwise.
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


def test_ep_world1_equals_single_device_and_oracle():
    from paper_2605_20179_b200 import tide
    layer = DeviceLayer(SHAPE, 41)
    desc = desc_for(SHAPE)
    ep = tide.EPContext(desc, tide.nccl_unique_id(), 0, 1)
    single = tide.Context(desc, SHAPE.num_experts)
    E, k = SHAPE.num_experts, SHAPE.top_k
    xs = g.block_hidden_np(SHAPE, 41)
    p_ep = torch.zeros(E, dtype=torch.uint8, device="cuda")
    p_1 = torch.zeros(E, dtype=torch.uint8, device="cuda")
    for t in range(SHAPE.steps):
        x = g.np_to_torch(xs[t], "cuda")
        r_ep = ep.moe_step_ep(x, layer.router, layer.device_all, shared_w=layer.shared,
                              placement=p_ep, step=t, interval=2, stats=True)
        r_1 = single.moe_step(x, layer.router, **layer.weights(), placement=p_1, step=t,
                              interval=2)
        torch.cuda.synchronize()
        assert torch.equal(r_ep.out.view(torch.int16), r_1.out.view(torch.int16)), t
        assert torch.equal(r_ep.hit_counts, r_1.hit_counts)
        assert torch.equal(r_ep.placement, r_1.placement)
        ref = oracle.moe_step(layer.oracle_layer(), xs[t], k, p_ep.cpu().numpy(), t, 2, E)
        assert (r_ep.hit_counts.cpu().numpy() == ref.hits).all()
        assert rel_err(to_np_f64(r_ep.out), ref.out) < OUT_TOL
        p_ep.copy_(r_ep.placement)
        p_1.copy_(r_1.placement)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _ep_rank(rank, world, port, q):
    import torch.distributed as dist
    from paper_2605_20179_b200 import tide
    try:
        torch.cuda.set_device(rank)
        os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        uid = [tide.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        layer = DeviceLayer(SHAPE, 42)
        desc = desc_for(SHAPE)
        ctx = tide.EPContext(desc, uid[0], rank, world, device=rank)
        E, k = SHAPE.num_experts, SHAPE.top_k
        El = E // world
        x_np = g.block_hidden_np(SHAPE, 300 + rank, steps=1)[0]
        r = ctx.moe_step_ep(g.np_to_torch(x_np, "cuda"), layer.router,
                            layer.device_all[rank * El:(rank + 1) * El].contiguous(),
                            shared_w=layer.shared,
                            placement=torch.zeros(El, dtype=torch.uint8, device="cuda"),
                            step=0, interval=1)
        torch.cuda.synchronize()
        ref = oracle.moe_step(layer.oracle_layer(), x_np, k, np.zeros(E, np.uint8), 0, 1, E)
        err = rel_err(to_np_f64(r.out), ref.out)
        # global hits = hits over all ranks' tokens
        tk = [None] * world
        dist.all_gather_object(tk, ref.topk_idx)
        hits_ok = bool((r.hit_counts.cpu().numpy() == oracle.hits(np.concatenate(tk), E)).all())
        q.put((rank, err, hits_ok))
        dist.destroy_process_group()
    except Exception as ex:
        q.put((rank, repr(ex), False))


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_ep_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ep_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
    for rank, err, hits_ok in res:
        assert not isinstance(err, str), err
        assert hits_ok and err < OUT_TOL, (rank, err)


def test_ep_wait_reports_completion():
    """tide_ctx_ep_wait (failure handling): returns once the last EP step completed, for the
    NCCL exchange (with ncclCommGetAsyncError polling) and the peer-memory exchange."""
    from paper_2605_20179_b200 import tide
    shape = g.Shape("epw", 32, 4, 256, 256, 1, 16, steps=2, dtype="bf16", shared_expert=True)
    layer = DeviceLayer(shape, 81)
    desc = desc_for(shape)
    nccl = tide.EPContext(desc, tide.nccl_unique_id(), 0, 1)
    p2p = tide.EPPeerContext(desc, 0, 1)
    p2p.connect(bases=[p2p.export()[1]])
    x = g.np_to_torch(g.block_hidden_np(shape, 81)[0], "cuda")
    for ctx in (nccl, p2p):
        ctx.wait(1000)  # no step yet: returns at once
        ctx.moe_step_ep(x, layer.router, layer.device_all, shared_w=layer.shared,
                        placement=torch.zeros(32, dtype=torch.uint8, device="cuda"), step=0,
                        interval=1)
        ctx.wait(20000)
