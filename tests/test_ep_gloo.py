"""Expert-parallel exchange protocol on CPU with torch.distributed gloo, world size 2.

The CUDA EP step (tide_moe_step_ep) moves bytes in this order: all-gather of every
rank's tokens and routing (fixed rows per rank) -> each rank computes its local experts
(e / (E/P) == rank) for every gathered row and sums g*y per source row in slot order ->
all-to-all of the per-source partials -> each rank sums the P partials in rank order;
global hits = all-gather of the local experts' counts (DESIGN R-18).  This test runs
exactly that dataflow with gloo collectives, the fp64 oracle supplying the per-expert
SwiGLU, and checks it against the single-device oracle step and the oracle's own EP
emulation (O11).  Test infrastructure only.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import tidegen as g

SHAPE = g.Shape("ep", 8, 3, 64, 64, 1, 6, steps=2, dtype="bf16")
P = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _rank_body(rank, world, q)
    except Exception as ex:  # report instead of hanging the parent
        q.put((rank, repr(ex), 0.0, False, False))
    finally:
        dist.destroy_process_group()


def _rank_body(rank, world, q):
    if True:
        lt = g.layer_np(SHAPE, 5)
        L = oracle.Layer(lt.wr, lt.wg, lt.wu, lt.wd)
        E, k, H = SHAPE.num_experts, SHAPE.top_k, SHAPE.hidden
        El = E // world
        x = g.block_hidden_np(SHAPE, 100 + rank, steps=1)[0]  # this rank's block
        N = x.shape[0]
        logits = oracle.router_logits(x, L.wr)
        topk = oracle.topk(logits, k)
        gates = oracle.gates(logits, topk, True)
        # dispatch: all-gather tokens (as float64 of the stored values), routing
        xs = torch.from_numpy(g.bf16_bits_to_f32(x).astype(np.float64))
        xs_all = [torch.empty_like(xs) for _ in range(world)]
        dist.all_gather(xs_all, xs)
        tk_all = [torch.empty(N, k, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(tk_all, torch.from_numpy(topk.astype(np.int64)))
        gt_all = [torch.empty(N, k, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gt_all, torch.from_numpy(gates))
        # local experts over every source row; partial sums per source row, slot order
        lo, hi = rank * El, (rank + 1) * El
        counts = np.zeros(El, np.int64)
        partial = torch.zeros(world, N, H, dtype=torch.float64)
        for p in range(world):
            for n in range(N):
                for j in range(k):
                    e = int(tk_all[p][n, j])
                    if lo <= e < hi:
                        counts[e - lo] += 1
                        y = oracle.swiglu(xs_all[p][n].numpy(), L.wg[e], L.wu[e], L.wd[e])
                        partial[p, n] += float(gt_all[p][n, j]) * torch.from_numpy(y)
        # combine: all-to-all of partials, rank-order sum
        recv = [torch.empty(N, H, dtype=torch.float64) for _ in range(world)]
        recv[rank] = partial[rank].clone()
        reqs = []  # all-to-all as point-to-point pairs (gloo has no alltoall)
        for p in range(world):
            if p != rank:
                reqs.append(dist.isend(partial[p].contiguous(), p))
                reqs.append(dist.irecv(recv[p], p))
        for r_ in reqs:
            r_.wait()
        out = recv[0].clone()
        for p in range(1, world):
            out += recv[p]
        hits_parts = [torch.empty(El, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(hits_parts, torch.from_numpy(counts))
        hits = torch.cat(hits_parts).numpy()
        # references
        single = oracle.moe_step(L, x, k, np.zeros(E, np.uint8), 0, 1, E)
        all_topk = np.concatenate([t.numpy() for t in tk_all]).astype(np.int32)
        q.put((rank, float(np.abs(out.numpy() - single.out).max()),
               float(np.abs(single.out).max()), bool((hits == oracle.hits(all_topk, E)).all()),
               bool((single.topk_idx == topk).all())))


def test_ep_protocol_world2_matches_single_device_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, P, port, q)) for r in range(P)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in range(P)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, err, scale, hits_ok, topk_ok in res:
        assert not isinstance(err, str), err
        assert topk_ok and hits_ok, rank
        assert err <= 1e-12 * max(scale, 1.0), (rank, err)


@pytest.mark.parametrize("shared", [False, True])
@pytest.mark.parametrize("P_", [2, 4])
def test_oracle_ep_emulation_matches_single_device(shared, P_):
    """O11 with P ranks on the same shapes (one process): EP moves bytes, not math, so it
    equals the single-device oracle step, shared expert (R-16) included."""
    sh = g.Shape("ep", 8, 3, 64, 64, 1, 6, steps=2, dtype="bf16", shared_expert=shared)
    lt = g.layer_np(sh, 5)
    L = oracle.Layer(lt.wr, lt.wg, lt.wu, lt.wd, lt.shared)
    x = g.block_hidden_np(sh, 100, steps=1)[0]
    E, k = sh.num_experts, sh.top_k
    single = oracle.moe_step(L, x, k, np.zeros(E, np.uint8), 0, 1, E)
    t, h, pout, out = oracle.ep_step(L, P_, x, k, np.zeros(E, np.uint8), 0, 1, E // P_)
    assert (h == single.hits).all() and pout.all()
    assert np.allclose(out, single.out, rtol=1e-13, atol=1e-14)
    if shared:  # the shared term is really there: dropping it changes the output
        L0 = oracle.Layer(lt.wr, lt.wg, lt.wu, lt.wd)
        assert not np.allclose(oracle.ep_step(L0, P_, x, k, np.zeros(E, np.uint8), 0, 1,
                                              E // P_)[3], out)
