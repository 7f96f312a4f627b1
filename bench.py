#!/usr/bin/env python
"""bench.py -- block-tokens/s per MoE layer-step of the TIDE hot path on B200.

One bench *step* = one denoising step of the block through every MoE layer of
the stack (20 layers for the mini config); each layer-step is the whole hot
path (router, top-k, hits, refresh/placement, permutation, grouped SwiGLU FFN
on tcgen05, combine; pinned-host serving when capacity < E), one
tide_moe_step call through the C ABI.

  value  = tokens x layer-steps / device time (CUDA events, max over ranks)
  e2e    = same metric with the block's hidden states H2D-copied from pinned
           host before, and the output D2H-copied after, every layer-step
  roofline = the grouped FFN kernel's algorithmic HBM bytes / its measured
           average launch time vs MEASURED_PEAKS.json hbm_gbs

`--impl reference` times the fp64 CPU oracle (the reference arm of this tier)
on a bounded sample of the same workload.  Multi-GPU (torchrun): every rank
runs its own blocks through its own replica of the stack (weak scaling, no
data-path collective); EP is listed in DESIGN.md as next.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import tidegen as g  # noqa: E402

METRIC = "block-tokens/sec per MoE layer-step"
UNIT = "block-tokens/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["tide", "reference"], default="tide")
    ap.add_argument("--config", choices=["mini", "sweep", "flash1"], default="mini")
    ap.add_argument("--capacity", type=int, default=0, help="0 = all experts in HBM (C = E)")
    ap.add_argument("--interval", type=int, default=4)
    ap.add_argument("--layers", type=int, default=0, help="override the stack depth")
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--routing", choices=["calibrated", "uniform"], default="calibrated",
                    help="calibrated temporal block routing (default) or the uniform iid stress "
                         "case (alpha=0, a0=0, skew=0: the most unique experts per launch)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=16.0)
    ap.add_argument("--eager", action="store_true",
                    help="launch every layer-step from the host in the timed region (default: "
                         "NEXT-3 CUDA graphs, one per block step t covering all layers)")
    ap.add_argument("--prefetch-mb", type=float, default=-1,
                    help="NEXT-3 cross-layer L2 prefetch budget per layer-step (MB); "
                         "-1 = default (32 MB when all experts are in HBM), 0 = off")
    ap.add_argument("--ep", action="store_true",
                    help="expert parallelism over the ranks (tide_moe_step_ep) instead of replicas")
    ap.add_argument("--p2p", action="store_true",
                    help="with --ep: dispatch/combine by the kernels over peer memory "
                         "(tide_ctx_create_ep_p2p) instead of NCCL collectives")
    return ap.parse_args()


def shape_for(args) -> g.Shape:
    if args.config == "mini":
        s = g.MINI
    elif args.config == "sweep":
        s = g.SWEEP
    else:  # one flash-shaped layer stack that fits HBM at C = E
        s = g.Shape("flash1", 256, 8, 4096, 1024, 8, 32)
    if args.layers:
        s = g.Shape(s.name, s.num_experts, s.top_k, s.hidden, s.ffn, args.layers, s.tokens,
                    s.steps, s.interval, s.capacity, s.dtype, s.shared_expert)
    return s


def workload_str(s: g.Shape, cap: int, interval: int) -> str:
    return (f"{s.name}: LLaDA2.0-{'mini' if s.hidden == 2048 else 'flash'}-shaped MoE stack, "
            f"{s.layers} layers, E={s.num_experts} top-{s.top_k}"
            f"{' + shared expert' if s.shared_expert else ''}, H={s.hidden}, F={s.ffn}, "
            f"{s.tokens} tokens per layer-step ({s.tokens // 32} block(s) of 32), "
            f"capacity {cap}{' (all experts in HBM)' if cap == s.num_experts else ' (pinned-host serving)'}, "
            f"refresh interval {interval}, T={s.steps} steps per block")


# ------------------------------------------------------------------ clocks
class Clocks:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        sm, mx, reasons = [], [], set()
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, v in zip(self.NAMES, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        os.unlink(self.f.name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "samples": len(sm),
                "reasons": sorted(reasons)}


# ------------------------------------------------------------------ oracle baseline
def oracle_rate(shape: g.Shape, seed: int, budget_s: float, tokens: int, threads: int,
                wt_host=None, routing: str = "calibrated"):
    """Time the fp64 CPU oracle (as it stands) on `threads` host threads, on full layer-steps
    of `tokens` tokens of layer 0, until `budget_s` seconds are spent."""
    import oracle
    uni = routing == "uniform"
    if wt_host is None:
        wr, wg, wu, wd, sh = g.layer_torch(shape, seed, 0, "cpu", skew=0.0 if uni else g.SKEW)
        to = g.torch_to_np
        wt_host = oracle.Layer(to(wr), to(wg), to(wu), to(wd),
                               tuple(to(a) for a in sh) if sh else None)
    xs = g.block_hidden_np(shape, seed, 0, steps=shape.steps, tokens=tokens, iid=uni)
    E = shape.num_experts
    oracle.set_threads(threads)
    used = oracle.get_threads()
    p = np.zeros(E, np.uint8)
    n_steps, t0 = 0, time.perf_counter()
    times = []
    while True:
        t = n_steps % shape.steps
        a = time.perf_counter()
        r = oracle.moe_step(wt_host, xs[t], shape.top_k, p, t, 4, E)
        times.append(time.perf_counter() - a)
        p = r.placement
        n_steps += 1
        if time.perf_counter() - t0 > budget_s:
            break
    el = sum(times)
    return {"value": round(tokens * n_steps / el, 3), "unit": UNIT, "cores": used,
            "kind": "oracle",
            "sample": f"{n_steps} full layer-steps (router..combine, fp64, {used} host thread(s), "
                      f"OpenMP over tokens) of layer 0, {tokens} tokens each, steps "
                      f"0..{n_steps - 1} of the block",
            "ms_per_layer_step": round(1e3 * el / n_steps, 3)}, wt_host


def cpu_baseline(shape: g.Shape, seed: int, budget_s: float, tokens: int, routing: str):
    """The oracle on every host core (the figure of record) and on one core, same sample."""
    ncores = os.cpu_count() or 1
    many, wt = oracle_rate(shape, seed, budget_s * 0.5, tokens, ncores, routing=routing)
    one, _ = oracle_rate(shape, seed, budget_s * 0.5, tokens, 1, wt_host=wt, routing=routing)
    many["single_thread"] = {k: one[k] for k in ("value", "cores", "sample", "ms_per_layer_step")}
    many["host_cpu"] = _cpu_model()
    return many


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip() + f" ({os.cpu_count()} logical CPUs)"
    except OSError:
        pass
    return f"{os.cpu_count()} logical CPUs"


# ------------------------------------------------------------------ main arm
def h2d_peak_gbs(dev, mb: int = 256, reps: int = 5) -> float:
    """Pinned-host -> HBM copy bandwidth (best of `reps` copies of `mb` MB, CUDA events):
    the PCIe roofline for the pinned-host serving path (a6, SURVEY 8(d) metric 4)."""
    src = torch.empty(mb << 20, dtype=torch.uint8).pin_memory()
    dst = torch.empty(mb << 20, dtype=torch.uint8, device=dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 0.0
    for _ in range(reps):
        a.record()
        dst.copy_(src, non_blocking=True)
        b.record()
        torch.cuda.synchronize()
        best = max(best, (mb << 20) / (a.elapsed_time(b) / 1e3) / 1e9)
    del src, dst
    return best


def max_over_ranks(v: float, world: int, dev) -> float:
    """MAX over ranks of a device-timed value (NCCL: device tensor; gloo test mode: host)."""
    if world == 1:
        return v
    gloo = torch.distributed.get_backend() == "gloo"
    tm = torch.tensor([v], device="cpu" if gloo else dev)
    torch.distributed.all_reduce(tm, op=torch.distributed.ReduceOp.MAX)
    return float(tm.item())


def run_tide(args, rank: int, world: int, local_rank: int):
    from paper_2605_20179_b200 import tide
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    s = shape_for(args)
    E, k, H, F, N, Lyr = s.num_experts, s.top_k, s.hidden, s.ffn, s.tokens, s.layers
    cap = args.capacity or E
    pool_mode = cap < E
    desc = tide.make_desc(E, k, H, F, N, tide.TIDE_BF16, shared_expert=s.shared_expert)
    seed = args.seed + 1000 * rank  # each rank runs its own blocks (weak scaling)
    ep = args.ep
    El = E // world if ep else E
    if ep:
        cap = min(args.capacity or El, El)
        pool_mode = False
        uid = [tide.nccl_unique_id() if rank == 0 else None]
        if world > 1:
            torch.distributed.broadcast_object_list(uid, src=0)

    # weights: generated on the device (bit-identical to the host generator), packed by the
    # product API (tide_pack_expert); one context per layer (EP: this rank's E/P experts)
    layers = []
    for l in range(Lyr):
        wr, wg, wu, wd, sh = g.layer_torch(s, args.seed, l, dev,
                                           skew=0.0 if args.routing == "uniform" else g.SKEW)
        if ep:
            sl = slice(rank * El, (rank + 1) * El)
            wg, wu, wd = wg[sl].contiguous(), wu[sl].contiguous(), wd[sl].contiguous()
        packed = tide.pack_layer(desc, wg, wu, wd)
        del wg, wu, wd
        torch.cuda.empty_cache()
        shared = torch.cat([a.reshape(-1) for a in sh]).contiguous() if sh else None
        w = {"device_all": packed} if not pool_mode else {"host_master": packed.cpu().pin_memory()}
        if pool_mode:
            del packed
        if ep and args.p2p:
            ctx = tide.EPPeerContext(desc, rank, world, local_rank)
            hs = [None] * world
            mine = ctx.export()
            if world > 1:
                torch.distributed.all_gather_object(hs, mine[0])
                ctx.connect(handles=hs)
                torch.distributed.barrier()
            else:
                ctx.connect(bases=[mine[1]])
        elif ep:
            ctx = tide.EPContext(desc, uid[0] if l == 0 else None, rank, world, local_rank,
                                 like=None if l == 0 else layers[0]["ctx"])
        else:
            ctx = tide.Context(desc, cap, 16, local_rank)
        layers.append(dict(router=wr, w=w, shared=shared, ctx=ctx,
                           x=g.block_hidden_torch(s, seed, l, dev, iid=args.routing == "uniform"),
                           pl=torch.zeros(El, dtype=torch.uint8, device=dev),
                           hits=torch.empty(E, dtype=torch.int32, device=dev),
                           out=torch.empty(N, H, dtype=torch.bfloat16, device=dev)))
    torch.cuda.synchronize()
    T = s.steps
    # NEXT-3: each layer prefetches the next layer's likely experts into L2 (ring: the
    # last layer prefetches layer 0 for the next step)
    pf_mb = args.prefetch_mb if args.prefetch_mb >= 0 else (32.0 if not pool_mode and not ep else 0.0)
    if pf_mb > 0 and not pool_mode and not ep:
        for li, L in enumerate(layers):
            nx = layers[(li + 1) % Lyr]
            L["ctx"].set_prefetch(nx["ctx"], nx["w"]["device_all"], int(pf_mb * 1e6))

    def layer_step(L, t, x=None, stats=False):
        xx = L["x"][t] if x is None else x
        if ep:
            return L["ctx"].moe_step_ep(xx, L["router"], L["w"]["device_all"],
                                        shared_w=L["shared"], placement=L["pl"], step=t,
                                        interval=args.interval, capacity=cap, out=L["out"],
                                        hit_counts=L["hits"], placement_out=L["pl"], stats=stats)
        return L["ctx"].moe_step(xx, L["router"], **L["w"],
                                 shared_w=L["shared"], placement=L["pl"], step=t,
                                 interval=args.interval, out=L["out"], hit_counts=L["hits"],
                                 placement_out=L["pl"], stats=stats)

    graphs = None

    def bench_step(i, eager=False):
        t = i % T
        if graphs is not None and not eager:
            graphs[t].replay()
            return
        for L in layers:
            layer_step(L, t)

    for i in range(args.warmup):
        bench_step(i)
    torch.cuda.synchronize()
    if not args.eager and not pool_mode and (not ep or args.p2p):  # NEXT-3: one graph per block step t, every layer-step of the stack in it
        gl = []
        for t in range(T):
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                for L in layers:
                    layer_step(L, t)
            gl.append(gr)
        torch.cuda.synchronize()
        graphs = gl
        for i in range(args.warmup):  # placement state continues from the eager warm-up
            bench_step(args.warmup + i)
        torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed_region(phase_timing: bool):
        for L in layers:
            L["ctx"].set_timing(phase_timing)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0.record(st)
        for i in range(args.steps):
            bench_step(args.warmup + i, eager=phase_timing)
        e1.record(st)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1)
        if world > 1:
            t = max_over_ranks(t, world, dev)
        ph = [L["ctx"].timing() for L in layers] if phase_timing else None
        for L in layers:
            L["ctx"].set_timing(False)
        return t, ph

    # region 1: the headline number (no per-phase events in the stream)
    clk = Clocks(local_rank)
    ms, _ = timed_region(False)
    clocks = clk.stop()
    # region 2: same steps with per-phase CUDA events on the launching stream (roofline)
    ms_phased, phases = timed_region(True)
    # region 3: each step timed alone (events between steps): refresh vs skipped steps
    # (SURVEY 8(d) metric 1; a step is a refresh step iff t % interval == 0)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    torch.cuda.synchronize()
    for i in range(args.steps):
        evs[i][0].record(st)
        bench_step(args.warmup + i)
        evs[i][1].record(st)
    torch.cuda.synchronize()
    per = [(a.elapsed_time(b), (args.warmup + i) % T % args.interval == 0)
           for i, (a, b) in enumerate(evs)]
    ref_ms = [m for m, r in per if r]
    skp_ms = [m for m, r in per if not r]
    step_split = {"ms_refresh_step": round(sum(ref_ms) / max(1, len(ref_ms)), 4),
                  "ms_skipped_step": round(sum(skp_ms) / max(1, len(skp_ms)), 4),
                  "refresh_steps": len(ref_ms), "skipped_steps": len(skp_ms),
                  "p50_ms_step": round(float(np.percentile([m for m, _ in per], 50)), 4),
                  "p90_ms_step": round(float(np.percentile([m for m, _ in per], 90)), 4)}
    layer_steps = args.steps * Lyr
    value = N * layer_steps * world / (ms / 1e3)

    # algorithmic FFN bytes of exactly the timed (layer, t) sequence: replay with stats
    # (untimed; routing is deterministic, so the same experts are hit)
    for L in layers:
        L["pl"].zero_()
    for i in range(args.warmup):
        for L in layers:
            layer_step(L, i % T)
    ffn_bytes, uniq, w_read, copies, h2d = 0, 0, 0, 0, 0
    R = N * k + (N if s.shared_expert else 0)
    act_bytes = R * (H * 2 + 2 * F * 2 + H * 4)
    for i in range(args.steps):
        for L in layers:
            r = layer_step(L, (args.warmup + i) % T, stats=True)
            u = r.stats["unique_experts"] + (1 if s.shared_expert else 0)
            uniq += u
            w_read += r.stats["weight_bytes_read"]
            if ep:  # this rank's local experts over every rank's rows
                pairs = r.stats["resident_pairs"] + r.stats["nonresident_pairs"]
                rows = pairs + (N if s.shared_expert else 0)
                ffn_bytes += u * s.expert_bytes + rows * (H * 2 + 2 * F * 2 + H * 4)
            else:
                ffn_bytes += u * s.expert_bytes + act_bytes
            copies += r.stats["copies"]
            h2d += r.stats["h2d_bytes"]
    ffn_ms = sum(p["ffn_ms"] for p in phases)
    ffn_launches = sum(p["ffn_launches"] for p in phases)
    launches = sum(p["launches"] for p in phases)
    tot = {kk: sum(p[kk] for p in phases) for kk in ("router_ms", "route_ms", "gather_ms",
                                                      "ffn_ms", "staged_ms", "combine_ms",
                                                      "total_ms")}
    # the resident FFN launch is one per layer-step: its bytes per launch
    per_launch_bytes = ffn_bytes / layer_steps
    ffn_avg_s = (tot["ffn_ms"] / 1e3) / layer_steps
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = peaks.get("hbm_gbs", 6650.0)
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else \
        "fallback 6.65 TB/s (B200_PROFILING.md)"
    achieved = per_launch_bytes / ffn_avg_s / 1e9
    traffic, traffic_detail = None, None
    tp = os.path.join(ROOT, "profiles", "ffn_traffic.json")
    if os.path.exists(tp):
        try:
            traffic_detail = json.load(open(tp)).get(s.name)
            traffic = traffic_detail["dram_bytes_per_launch"] if traffic_detail else None
        except Exception:
            traffic, traffic_detail = None, None
    flops_per_layer_step = 2 * N * k * 3 * H * F + (2 * N * 3 * H * F if s.shared_expert else 0)
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "frac_of_nominal_8TBps": round(achieved / 8000.0, 4),
                "traffic_detail": traffic_detail,
                "kernel": "tide_ffn_kernel (grouped SwiGLU, tcgen05 + TMA)",
                "peak_source": peak_src,
                "bytes_per_launch": round(per_launch_bytes),
                "avg_launch_us": round(ffn_avg_s * 1e6, 2),
                "ffn_share_of_step": round(tot["ffn_ms"] / max(tot["total_ms"], 1e-9), 4),
                "tensor_frac": round(flops_per_layer_step / ffn_avg_s / 1e12 /
                                     peaks.get("bf16_tflops", 1590.0), 5),
                "unique_experts_per_layer_step": round(uniq / layer_steps, 2)}

    # e2e: hidden states from pinned host in, output to pinned host out, every layer-step
    e2e = None
    if not args.no_e2e:
        Ly = len(layers)
        # inputs of step t for every layer contiguous in pinned host memory: layer 0's input
        # goes first, layers 1.. in one copy that lands while layer 0 computes
        xh = torch.stack([L["x"] for L in layers], 1).cpu().pin_memory()  # [T, L, N, H]
        oh = [torch.empty(N, H, dtype=torch.bfloat16).pin_memory() for _ in layers]
        xd = torch.empty(Ly, N, H, dtype=torch.bfloat16, device=dev)
        cs = torch.cuda.Stream(device=dev)  # copy stream: PCIe transfers overlap the layer-steps
        ev_in = [torch.cuda.Event(), torch.cuda.Event()]
        ev_out = [torch.cuda.Event() for _ in layers]

        def e2e_step(t):
            # the step's inputs go H2D on the copy stream (after the previous step's compute has
            # consumed the buffers); each layer-step's output goes D2H on the copy stream while
            # the next layer-step runs
            ms = torch.cuda.current_stream()  # the capture stream under torch.cuda.graph
            cs.wait_stream(ms)
            with torch.cuda.stream(cs):
                xd[0].copy_(xh[t, 0], non_blocking=True)
                ev_in[0].record(cs)
                if Ly > 1:
                    xd[1:].copy_(xh[t, 1:], non_blocking=True)
                    ev_in[1].record(cs)
            for li, L in enumerate(layers):
                if li < 2:
                    ms.wait_event(ev_in[li])
                layer_step(L, t, x=xd[li])
                ev_out[li].record(ms)
                cs.wait_event(ev_out[li])
                with torch.cuda.stream(cs):
                    oh[li].copy_(L["out"], non_blocking=True)
            ms.wait_stream(cs)

        e2e_graphs = None
        if graphs is not None:  # same launch mode as the headline: copies captured in the graphs
            e2e_graphs = []
            for t in range(T):
                gr = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gr):
                    e2e_step(t)
                e2e_graphs.append(gr)
            for i in range(args.warmup):
                e2e_graphs[(args.warmup + i) % T].replay()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0.record(st)
        for i in range(args.steps):
            t = (args.warmup + i) % T
            if e2e_graphs is not None:
                e2e_graphs[t].replay()
            else:
                e2e_step(t)
        e1.record(st)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        if world > 1:
            ems = max_over_ranks(ems, world, dev)
        e2e = {"value": N * layer_steps * world / (ems / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": Lyr * N * H * 2, "d2h_bytes_per_step": Lyr * N * H * 2,
               "ms_per_step": ems / args.steps,
               "launch": "CUDA graph per block step (copies captured)" if e2e_graphs else "eager",
               "note": "tide_moe_step through the C ABI; per layer-step the block's hidden "
                       "states are copied from pinned host and the output back, on a copy "
                       "stream that overlaps the transfers with the layer-steps"}
        del e2e_graphs

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:  # the CPU baseline is an N=1 figure
        cpu = cpu_baseline(s, args.seed, args.cpu_seconds, min(N, 32), args.routing)

    io = None
    if pool_mode:  # a6: the H2D link is the roofline of capacity-limited steps
        pk = h2d_peak_gbs(dev)
        eff = (h2d / args.steps) / (ms / args.steps / 1e3) / 1e9
        io = {"copies_per_step": copies / args.steps, "h2d_bytes_per_step": h2d / args.steps,
              "h2d_gbs_effective": round(eff, 2), "h2d_peak_gbs": round(pk, 2),
              "frac": round(eff / pk, 4),
              "note": "effective = expert bytes copied H2D per step / device time per step; "
                      "peak = best pinned-host -> HBM copy of 256 MB measured in this run"}
    res = {"metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
           "data": "synthetic: tidegen seeded weights (U(+-sqrt(3/fan_in)), bf16) and " +
                   ("calibrated temporal block routing (alpha=0.99, skew=0.5, a0=0.8)"
                    if args.routing == "calibrated" else
                    "uniform iid stress routing (alpha=0, a0=0, skew=0)"),
           "config": {"workload": workload_str(s, cap, args.interval), "layers": Lyr,
                      "tokens_per_layer_step": N, "num_experts": E, "top_k": k, "hidden": H,
                      "ffn": F, "capacity": cap, "interval": args.interval,
                      "routing": args.routing,
                      "parallelism": (f"expert parallel x{world} (E/P = {El} experts per rank, "
                                      + ("peer-memory dispatch/combine kernels)" if args.p2p else
                                         "NCCL all-gather dispatch + all-to-all combine)")) if ep
                      else f"replicas x{world} (each rank its own blocks)",
                      "l2": "inputs larger than L2: each layer's weights (>=1.6 GB) rotate "
                            "through the stack between reuses",
                      "launch": ("CUDA graph per block step (all layers), replayed" if graphs
                                 else "eager stream (PDL-chained kernels)"),
                      "prefetch_mb": pf_mb},
           "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
           "gpu_launches": launches * world if rank == 0 else launches,
           "clocks": clocks,
           "phases_us_per_layer_step": {kk: round(1e3 * v / layer_steps, 2) for kk, v in tot.items()},
           "ms_per_step_with_phase_events": round(ms_phased / args.steps, 4),
           "step_split": step_split,
           "io": io}
    return res


def run_reference(args):
    """Reference arm of this tier: the fp64 CPU oracle, as it stands, timed on every host core
    (OpenMP over tokens) on the bench workload's layer-steps (layer 0 of the stack, the
    block's full token count)."""
    import oracle
    s = shape_for(args)
    N = s.tokens
    uni = args.routing == "uniform"
    wr, wg, wu, wd, sh = g.layer_torch(s, args.seed, 0, "cpu", skew=0.0 if uni else g.SKEW)
    to = g.torch_to_np
    L = oracle.Layer(to(wr), to(wg), to(wu), to(wd), tuple(to(a) for a in sh) if sh else None)
    xs = g.block_hidden_np(s, args.seed, 0, steps=s.steps, tokens=N, iid=uni)
    E = s.num_experts
    cap = args.capacity or E
    oracle.set_threads(os.cpu_count() or 1)
    cores = oracle.get_threads()
    p = np.zeros(E, np.uint8)
    for i in range(args.warmup):
        p = oracle.moe_step(L, xs[i % s.steps], s.top_k, p, i % s.steps, args.interval, cap).placement
    t0 = time.perf_counter()
    for i in range(args.steps):
        t = (args.warmup + i) % s.steps
        p = oracle.moe_step(L, xs[t], s.top_k, p, t, args.interval, cap).placement
    el = time.perf_counter() - t0
    v = N * args.steps / el
    sample = (f"each step = one full layer-step (router..combine, fp64, {cores} host threads, "
              f"OpenMP over tokens) of layer 0 of the stack on all {N} tokens of the block")
    return {"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": UNIT,
            "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * el / args.steps, 2), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_str(s, cap, args.interval), "layers": s.layers,
                       "tokens_per_layer_step": s.tokens, "num_experts": E, "top_k": s.top_k,
                       "hidden": s.hidden, "ffn": s.ffn, "capacity": cap,
                       "interval": args.interval, "routing": args.routing,
                       "oracle_sample": f"layer 0 of {s.layers}, all {N} tokens per step"},
            "cpu_baseline": {"value": round(v, 3), "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": sample, "host_cpu": _cpu_model()},
            "e2e": {"value": round(v, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # test mode for the multi-process code path on a one-GPU box: every rank on cuda:0 and a
    # gloo process group (NCCL refuses two ranks on one device); only --ep --p2p and replicas
    if os.environ.get("TIDE_BENCH_SAME_DEVICE"):
        local_rank = 0
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args)), flush=True)
        return
    if world > 1:
        torch.cuda.set_device(local_rank)
        if os.environ.get("TIDE_BENCH_SAME_DEVICE"):
            torch.distributed.init_process_group("gloo")
        else:
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    res = run_tide(args, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
