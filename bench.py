#!/usr/bin/env python
"""bench.py -- block-tokens/s per MoE layer-step of the TIDE hot path on B200.

One bench *step* = one denoising step of the block(s) through every MoE layer of the
stack; each layer-step is the whole hot path (router, top-k, hits, refresh/placement,
permutation, grouped SwiGLU FFN on tcgen05, combine; pinned-host serving when
capacity < E; the expert-parallel exchange under EP), one tide_moe_step /
tide_moe_step_ep call through the C ABI.

  value    = tokens x layer-steps, summed over ranks / device time (CUDA events, max over
             ranks)
  e2e      = same metric with every layer-step's hidden states H2D-copied from pinned host
             and its output D2H-copied, inside the timed region
  roofline = the dominant kernel's algorithmic bytes / its measured launch time vs
             MEASURED_PEAKS.json (the grouped FFN and HBM when every expert is in HBM; the
             H2D link when capacity < E)

N = 1 (default): BJ.configs[1] (mini stack, C = E) is the headline; `sub_results` adds the
8-block sweep batch (BJ.configs[4], C = E) and the flash-shaped stack with pinned-host
serving at the paper's budget C = 64 and at C = 217 (BJ.configs[2], 8 of 32 layers: the
full stack does not fit one GPU).
N > 1 (`--gpus N`, spawned through torchrun when WORLD_SIZE is unset): BJ.configs[3], the
flash-shaped 32-layer stack expert-parallel over the N GPUs (E/N experts per rank, all in
HBM), one block per rank (weak scaling), dispatch/combine inside the kernels over peer
memory (NVLink); the NCCL all-gather / all-to-all variant is reported beside it.
`--replicas` runs independent per-rank stacks instead.

`--impl reference` times the fp64 CPU oracle (the reference arm of this tier) on every host
core on the same workload's layer-steps.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
NVLINK_GBS = 900.0  # NVLink 5 per direction per GPU (SURVEY 8(d) metric 5)
PAPER_CONTEXT = {
    "note": "The paper's published numbers are end-to-end dLLM decode speed-ups of its GPU-CPU "
            "system over baselines, on other hardware and with real LLaDA2.0 weights; they are "
            "context, not a target for this layer-step metric (vs_baseline is null).",
    "speedup_vs_best_baseline": "1.4x (LLaDA2.0-mini) / 1.5x (LLaDA2.0-flash) decode throughput "
                                "(P:14, P:440)",
    "hardware": "NVIDIA A100 80GB and H100 80GB + host CPU (48-core), PCIe (P:350)",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["tide", "reference"], default="tide")
    ap.add_argument("--config", choices=["mini", "sweep", "flash1", "flash"], default=None,
                    help="default: mini at N=1, flash (expert parallel) at N>1")
    ap.add_argument("--capacity", type=int, default=0, help="0 = all experts in HBM (C = E)")
    ap.add_argument("--interval", type=int, default=4)
    ap.add_argument("--layers", type=int, default=0, help="override the stack depth")
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--routing", choices=["calibrated", "uniform"], default="calibrated",
                    help="calibrated temporal block routing (default) or the uniform iid stress "
                         "case (alpha=0, a0=0, skew=0: the most unique experts per launch)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sub", action="store_true", help="skip the sub-results")
    ap.add_argument("--cpu-seconds", type=float, default=16.0)
    ap.add_argument("--eager", action="store_true",
                    help="launch every layer-step from the host in the timed region (default: "
                         "NEXT-3 CUDA graphs, one per block step t covering all layers)")
    ap.add_argument("--prefetch-mb", type=float, default=-1,
                    help="NEXT-3 cross-layer L2 prefetch budget per layer-step (MB); "
                         "-1 = default (32 MB when all experts are in HBM), 0 = off")
    ap.add_argument("--h2d-prefetch", type=int, default=0,
                    help="NEXT-3 H2D prefetch with pinned-host serving: experts per layer copied "
                         "ahead into the next layer's prefetch slots (0 = off)")
    ap.add_argument("--ep", action="store_true",
                    help="expert parallelism over the ranks (default at N>1; also at N=1)")
    ap.add_argument("--p2p", action="store_true",
                    help="with --ep at N=1: dispatch/combine by the kernels over peer memory "
                         "(the N>1 default)")
    ap.add_argument("--nccl", action="store_true",
                    help="EP headline on the NCCL collectives instead of peer memory")
    ap.add_argument("--strong", action="store_true",
                    help="EP strong scaling (SURVEY 8(d) flash-EP): 8 blocks (256 tokens) in "
                         "total per layer-step, split over the N ranks (default: one block "
                         "per rank, weak scaling)")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: independent per-rank stacks (no data-path collective) instead of EP")
    return ap.parse_args()


SHAPES = {"mini": g.MINI, "sweep": g.SWEEP, "flash": g.FLASH,
          "flash1": g.Shape("flash1", 256, 8, 4096, 1024, 8, 32)}


def shape_for(name: str, layers: int = 0) -> g.Shape:
    s = SHAPES[name]
    if layers:
        s = g.Shape(s.name, s.num_experts, s.top_k, s.hidden, s.ffn, layers, s.tokens,
                    s.steps, s.interval, s.capacity, s.dtype, s.shared_expert)
    return s


def workload_str(s: g.Shape, cap: int, interval: int, ep_world: int = 0) -> str:
    kind = "mini" if s.hidden == 2048 else "flash"
    if ep_world:
        where = (f"expert parallel over {ep_world} GPU(s), {s.num_experts // ep_world} experts "
                 f"per rank, capacity {cap} per rank")
    else:
        where = (f"capacity {cap}" + (" (all experts in HBM)" if cap == s.num_experts
                                      else " (pinned-host serving)"))
    return (f"{s.name}: LLaDA2.0-{kind}-shaped MoE stack, {s.layers} layers, E={s.num_experts} "
            f"top-{s.top_k}{' + shared expert' if s.shared_expert else ''}, H={s.hidden}, "
            f"F={s.ffn}, {s.tokens} tokens per layer-step per rank ({s.tokens // 32} block(s) "
            f"of 32), {where}, refresh interval {interval}, T={s.steps} steps per block")


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
                                       "--format=csv,noheader,nounits", "-lms", "50"],
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


# ------------------------------------------------------------------ helpers
def h2d_peak_gbs(dev, mb: int = 256, reps: int = 5) -> float:
    """Pinned-host -> HBM copy bandwidth (best of `reps` copies of `mb` MB, CUDA events):
    the PCIe roofline for the pinned-host serving path (a6, SURVEY 8(d) metric 4)."""
    torch.cuda.synchronize()  # no copy of the run (e.g. an H2D prefetch) shares the link
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


def reduce_over_ranks(v: float, world: int, dev, op="max") -> float:
    """MAX (or MIN) over ranks of a device-timed value (NCCL: device tensor; gloo: host)."""
    if world == 1:
        return v
    gloo = torch.distributed.get_backend() == "gloo"
    tm = torch.tensor([v], dtype=torch.float64, device="cpu" if gloo else dev)
    torch.distributed.all_reduce(tm, op=torch.distributed.ReduceOp.MAX if op == "max"
                                 else torch.distributed.ReduceOp.MIN)
    return float(tm.item())


def gather_over_ranks(vec: list, world: int, dev) -> list:
    if world == 1:
        return [list(vec)]
    gloo = torch.distributed.get_backend() == "gloo"
    t = torch.tensor(vec, dtype=torch.float64, device="cpu" if gloo else dev)
    out = [torch.empty_like(t) for _ in range(world)]
    torch.distributed.all_gather(out, t)
    return [o.cpu().tolist() for o in out]


def gather_tensor(t: torch.Tensor, world: int, dev) -> list:
    """All ranks' copies of a same-shape device tensor (NCCL: on the device; gloo: via host)."""
    if world == 1:
        return [t]
    gloo = torch.distributed.get_backend() == "gloo"
    src = t.contiguous().cpu() if gloo else t.contiguous()
    out = [torch.empty_like(src) for _ in range(world)]
    torch.distributed.all_gather(out, src)
    return [o.to(dev) for o in out]


def ep_check(st, args, s: g.Shape, dev, rank: int, world: int, p2p: bool) -> dict:
    """Correctness of the measured EP configuration on this machine, checked on the GPU: one
    EP layer-step (layer 0, t = 0) on every rank's tokens against the single-device step over
    all ranks' tokens, computed on rank 0 with every expert of the layer (DESIGN 8: the
    peer-memory EP output is bitwise equal to it for any world size; the NCCL path sums the
    ranks' partials in rank order, so it is compared within the 2e-2 output tolerance)."""
    tide = st.tide
    L = st.layers[0]
    st.reset()
    st.layer_step(L, 0)
    torch.cuda.synchronize()
    xs = gather_tensor(L["x"][0], world, dev)
    outs = gather_tensor(L["out"], world, dev)
    res = torch.zeros(3, dtype=torch.float64, device=dev)
    if rank == 0:
        E, k, H, F = s.num_experts, s.top_k, s.hidden, s.ffn
        x = torch.cat(xs)
        desc = tide.make_desc(E, k, H, F, x.shape[0], tide.TIDE_BF16, shared_expert=s.shared_expert)
        _, w, shared = gen_layer(args, s, 0, dev, desc)  # every expert of layer 0
        ctx = tide.Context(desc, E, 16, dev.index)
        pl = torch.zeros(E, dtype=torch.uint8, device=dev)
        r = ctx.moe_step(x, L["router"], device_all=w, shared_w=shared, placement=pl, step=0,
                         interval=args.interval)
        torch.cuda.synchronize()
        ep_out = torch.cat(outs)
        diff = (r.out.view(torch.int16) != ep_out.view(torch.int16)).sum()
        ref = r.out.float()
        rel = (ep_out.float() - ref).abs().max() / ref.abs().max().clamp_min(1e-30)
        res[0], res[1], res[2] = float(diff.item()), float(rel.item()), float(x.shape[0])
        ctx.close()
        del w, shared, ctx, r
        torch.cuda.empty_cache()
    if world > 1:
        gloo = torch.distributed.get_backend() == "gloo"
        rr = res.cpu() if gloo else res
        torch.distributed.broadcast(rr, 0)
        res = rr
    mism, rel, ntok = int(res[0].item()), float(res[1].item()), int(res[2].item())
    return {"layer": 0, "step": 0, "tokens": ntok, "mismatched_elements": mism,
            "bitwise_equal_single_device": mism == 0, "max_rel_err": rel,
            "pass": (mism == 0) if p2p else rel < 2e-2,
            "how": "rank 0 recomputes the layer-step over all ranks' tokens on one GPU with "
                   "every expert and compares the gathered EP outputs"}


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def traffic_for(key: str):
    """ncu DRAM bytes per FFN launch for exactly this run configuration, else None."""
    tp = os.path.join(ROOT, "profiles", "ffn_traffic.json")
    try:
        d = json.load(open(tp)).get(key)
    except Exception:
        return None, None
    return (d["dram_bytes_per_launch"], d) if d else (None, None)


def act_bytes(H, F, rows):
    """Per FFN row: x gathered (2H) + h written and read (2*2F) + y written (4H)."""
    return rows * (H * 2 + 2 * F * 2 + H * 4)


def gen_layer(args, s: g.Shape, l: int, dev, desc, experts=None, host=False):
    """One layer's (router, packed experts, packed shared expert) from the seeded generator,
    packed by the product API (tide_pack_expert); `host` moves the experts to pinned host."""
    from paper_2605_20179_b200 import tide
    wr, wg, wu, wd, sh = g.layer_torch(s, args.seed, l, dev,
                                       skew=0.0 if args.routing == "uniform" else g.SKEW,
                                       experts=experts)
    packed = tide.pack_layer(desc, wg, wu, wd)
    del wg, wu, wd
    shared = torch.cat([a.reshape(-1) for a in sh]).contiguous() if sh else None
    if host:
        hm = packed.cpu().pin_memory()
        del packed
        packed = hm
    torch.cuda.empty_cache()
    return wr, packed, shared


# ------------------------------------------------------------------ the stack
class Stack:
    """One rank's MoE stack: per layer a context, weights, router, inputs for T steps.
    mode: device_all | host_master | ep."""

    def __init__(self, args, s: g.Shape, dev, rank: int, world: int, cap: int, mode: str,
                 weights=None, p2p=False):
        from paper_2605_20179_b200 import tide
        self.tide, self.args, self.s, self.dev = tide, args, s, dev
        self.rank, self.world, self.mode, self.p2p = rank, world, mode, p2p
        E, k, H, F, N = s.num_experts, s.top_k, s.hidden, s.ffn, s.tokens
        self.El = E // world if mode == "ep" else E
        self.cap = cap
        self.desc = tide.make_desc(E, k, H, F, N, tide.TIDE_BF16, shared_expert=s.shared_expert)
        uni = args.routing == "uniform"
        seed_x = args.seed + 1000 * rank  # each rank runs its own blocks (weak scaling)
        self.layers = []
        for l in range(s.layers):
            if weights is not None:
                wr, w, shared = weights[l]
            else:
                ids = range(rank * self.El, (rank + 1) * self.El) if mode == "ep" else None
                wr, w, shared = gen_layer(args, s, l, dev, self.desc, ids,
                                          host=mode == "host_master")
            if mode == "ep" and p2p:
                ctx = tide.EPPeerContext(self.desc, rank, world, dev.index)
            elif mode == "ep":
                first = self.layers[0]["ctx"] if l else None
                uid = None
                if first is None:
                    uid = [tide.nccl_unique_id() if rank == 0 else None]
                    if world > 1:
                        torch.distributed.broadcast_object_list(uid, src=0)
                    uid = uid[0]
                ctx = tide.EPContext(self.desc, uid, rank, world, dev.index, like=first)
            else:
                ctx = tide.Context(self.desc, cap, 16, dev.index)
            self.layers.append(dict(router=wr, w=w, shared=shared, ctx=ctx,
                                    x=g.block_hidden_torch(s, seed_x, l, dev, iid=uni),
                                    pl=torch.zeros(self.El, dtype=torch.uint8, device=dev),
                                    hits=torch.empty(E, dtype=torch.int32, device=dev),
                                    out=torch.empty(N, H, dtype=torch.bfloat16, device=dev)))
        if mode == "ep" and p2p:
            self._connect()
        torch.cuda.synchronize()
        self.graphs = None

    def weights(self):
        return [(L["router"], L["w"], L["shared"]) for L in self.layers]

    def _connect(self):
        for L in self.layers:
            ctx = L["ctx"]
            h, base = ctx.export()
            if self.world > 1:
                hs = [None] * self.world
                torch.distributed.all_gather_object(hs, h)
                ctx.connect(handles=hs)
            else:
                ctx.connect(bases=[base])
        if self.world > 1:
            torch.distributed.barrier()

    def set_prefetch(self, mb: float):
        Ly = len(self.layers)
        for li, L in enumerate(self.layers):
            nx = self.layers[(li + 1) % Ly]
            L["ctx"].set_prefetch(nx["ctx"] if mb > 0 else None, nx["w"] if mb > 0 else None,
                                  int(mb * 1e6))

    def set_h2d_prefetch(self, n_experts: int):
        """NEXT-3 H2D prefetch (pinned-host serving): each layer's step copies the next
        layer's predicted streamed experts into that layer's prefetch slots."""
        Ly = len(self.layers)
        for li, L in enumerate(self.layers):
            nx = self.layers[(li + 1) % Ly]
            L["ctx"].set_prefetch(nx["ctx"], None, n_experts * self.s.expert_bytes)

    def layer_step(self, L, t, x=None, stats=False):
        xx = L["x"][t] if x is None else x
        a = self.args
        if self.mode == "ep":
            return L["ctx"].moe_step_ep(xx, L["router"], L["w"], shared_w=L["shared"],
                                        placement=L["pl"], step=t, interval=a.interval,
                                        capacity=self.cap, out=L["out"], hit_counts=L["hits"],
                                        placement_out=L["pl"], stats=stats)
        wk = {"device_all": L["w"]} if self.mode == "device_all" else {"host_master": L["w"]}
        return L["ctx"].moe_step(xx, L["router"], **wk, shared_w=L["shared"], placement=L["pl"],
                                 step=t, interval=a.interval, out=L["out"], hit_counts=L["hits"],
                                 placement_out=L["pl"], stats=stats)

    def step(self, i, eager=False):
        t = i % self.s.steps
        if self.graphs is not None and not eager:
            self.graphs[t].replay()
            return
        for L in self.layers:
            self.layer_step(L, t)

    def reset(self):
        for L in self.layers:
            L["pl"].zero_()

    def capture(self, warmup):
        """NEXT-3: one CUDA graph per block step t, every layer-step of the stack in it."""
        gl = []
        for t in range(self.s.steps):
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                for L in self.layers:
                    self.layer_step(L, t)
            gl.append(gr)
        torch.cuda.synchronize()
        self.graphs = gl
        for i in range(warmup):  # placement state continues from the eager warm-up
            self.step(warmup + i)
        torch.cuda.synchronize()

    def timed(self, steps, warmup, phase_timing=False):
        for L in self.layers:
            L["ctx"].set_timing(phase_timing)
        if self.world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for i in range(steps):
            self.step(warmup + i, eager=phase_timing)
        e1.record(st)
        torch.cuda.synchronize()
        ms = reduce_over_ranks(e0.elapsed_time(e1), self.world, self.dev)
        ph = [L["ctx"].timing() for L in self.layers] if phase_timing else None
        for L in self.layers:
            L["ctx"].set_timing(False)
        return ms, ph

    def step_split(self, steps, warmup):
        """Each step timed alone: refresh (t % interval == 0) vs skipped steps (8(d) metric 1)."""
        st = torch.cuda.current_stream()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(steps)]
        torch.cuda.synchronize()
        for i in range(steps):
            evs[i][0].record(st)
            self.step(warmup + i)
            evs[i][1].record(st)
        torch.cuda.synchronize()
        per = [(a.elapsed_time(b), (warmup + i) % self.s.steps % self.args.interval == 0)
               for i, (a, b) in enumerate(evs)]
        ref = [m for m, r in per if r]
        skp = [m for m, r in per if not r]
        return {"ms_refresh_step": round(sum(ref) / max(1, len(ref)), 4),
                "ms_skipped_step": round(sum(skp) / max(1, len(skp)), 4),
                "refresh_steps": len(ref), "skipped_steps": len(skp),
                "p50_ms_step": round(float(np.percentile([m for m, _ in per], 50)), 4),
                "p90_ms_step": round(float(np.percentile([m for m, _ in per], 90)), 4)}

    def stats_replay(self, steps, warmup):
        """Replay exactly the timed (layer, t) sequence eagerly with stats (untimed; routing is
        deterministic, so the same experts are hit) -> per-launch algorithmic bytes."""
        s = self.s
        self.reset()
        for i in range(warmup):
            for L in self.layers:
                self.layer_step(L, i % s.steps)
        acc = dict(alg=0, res_alg=0, uniq=0, copies=0, h2d=0, streamed=0, launches=0)
        sh = 1 if s.shared_expert else 0
        for i in range(steps):
            for L in self.layers:
                r = self.layer_step(L, (warmup + i) % s.steps, stats=True).stats
                u = r["unique_experts"] + sh
                acc["uniq"] += u
                rows_all = r["resident_pairs"] + r["nonresident_pairs"] + (s.tokens if sh else 0)
                acc["alg"] += u * s.expert_bytes + act_bytes(s.hidden, s.ffn, rows_all)
                # resident launch: hit experts whose weights were in HBM at step start (+ shared)
                acc["res_alg"] += ((u - r["experts_streamed"]) * s.expert_bytes
                                   + act_bytes(s.hidden, s.ffn, r["resident_rows"]))
                acc["copies"] += r["copies"]
                acc["h2d"] += r["h2d_bytes"]
                acc["streamed"] += r["experts_streamed"]
                acc["launches"] += r["ffn_launches"]
        return acc

    def routing_stats(self, B=64):
        """the routing the synthetic inputs produce, measured on the GPU's own
        routing over one block of layer 0 with the NEXT-4 analytics kernel (tide_trace_stats):
        mean adjacent-step and lag-5 cosine of the hit-count vectors, unique
        experts per step, mean Eq. 4 drift of the top-B placement."""
        s, L = self.s, self.layers[0]
        T = s.steps
        counts = torch.empty(T, s.num_experts, dtype=torch.int32, device=self.dev)
        self.reset()
        for t in range(T):
            self.layer_step(L, t)
            counts[t].copy_(L["hits"])
        sim, uq, dr = self.tide.trace_stats(counts, min(B, s.num_experts))
        torch.cuda.synchronize()
        sim = sim.cpu().numpy()
        uq = uq.cpu().numpy()
        return {"adjacent_cosine": round(float(np.mean([sim[t, t + 1] for t in range(T - 1)])), 4),
                "lag5_cosine": round(float(np.mean([sim[t, t + 5] for t in range(T - 5)])), 4),
                "unique_experts_per_step": [int(v) for v in uq],
                "drift_top%d_mean" % min(B, s.num_experts): round(float(dr.cpu().numpy().mean()), 4),
                "paper": "adjacent 0.985 (P:200), > 0.95 at 5 steps (P:203), unique experts grow "
                         "within a block (P:126-127)",
                "layer": 0}

    def e2e(self, steps, warmup, graphs: bool):
        """Same metric through the public API with every layer-step's hidden states copied
        H2D from pinned host and its output D2H, on a copy stream that overlaps the transfers
        with the layer-steps; captured in per-step graphs like the headline when it uses them."""
        s, dev = self.s, self.dev
        N, H = s.tokens, s.hidden
        Ly = len(self.layers)
        xh = torch.stack([L["x"] for L in self.layers], 1).cpu().pin_memory()  # [T, L, N, H]
        oh = [torch.empty(N, H, dtype=torch.bfloat16).pin_memory() for _ in self.layers]
        xd = torch.empty(Ly, N, H, dtype=torch.bfloat16, device=dev)
        cs = torch.cuda.Stream(device=dev)
        ev_in = [torch.cuda.Event(), torch.cuda.Event()]
        ev_out = [torch.cuda.Event() for _ in self.layers]

        def e2e_step(t):
            ms = torch.cuda.current_stream()
            cs.wait_stream(ms)
            with torch.cuda.stream(cs):
                xd[0].copy_(xh[t, 0], non_blocking=True)
                ev_in[0].record(cs)
                if Ly > 1:
                    xd[1:].copy_(xh[t, 1:], non_blocking=True)
                    ev_in[1].record(cs)
            for li, L in enumerate(self.layers):
                if li < 2:
                    ms.wait_event(ev_in[li])
                self.layer_step(L, t, x=xd[li])
                ev_out[li].record(ms)
                cs.wait_event(ev_out[li])
                with torch.cuda.stream(cs):
                    oh[li].copy_(L["out"], non_blocking=True)
            ms.wait_stream(cs)

        gl = None
        if graphs:
            gl = []
            for t in range(s.steps):
                gr = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gr):
                    e2e_step(t)
                gl.append(gr)
            for i in range(warmup):
                gl[(warmup + i) % s.steps].replay()
        if self.world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for i in range(steps):
            t = (warmup + i) % s.steps
            if gl is not None:
                gl[t].replay()
            else:
                e2e_step(t)
        e1.record(st)
        torch.cuda.synchronize()
        ems = reduce_over_ranks(e0.elapsed_time(e1), self.world, dev)
        del gl
        return {"value": round(N * steps * Ly * self.world / (ems / 1e3), 1), "unit": UNIT,
                "h2d_bytes_per_step": Ly * N * H * 2, "d2h_bytes_per_step": Ly * N * H * 2,
                "ms_per_step": round(ems / steps, 4),
                "launch": "CUDA graph per block step (copies captured)" if graphs else "eager",
                "note": "per layer-step the block's hidden states are copied from pinned host "
                        "and the output back (per rank), on a copy stream that overlaps the "
                        "transfers with the layer-steps"}

    def close(self):
        self.graphs = None
        for L in self.layers:
            L["ctx"].close()


def phase_sums(phases):
    keys = ("router_ms", "route_ms", "gather_ms", "ffn_ms", "staged_ms", "combine_ms", "total_ms")
    return {kk: sum(p[kk] for p in phases) for kk in keys}, sum(p["launches"] for p in phases)


# ------------------------------------------------------------------ single device
def measure_single(args, s: g.Shape, cap: int, dev, rank=0, world=1, weights=None, full=True,
                   steps=None, warmup=None, h2d_prefetch=None):
    """One single-device (or replica) run of stack `s` at capacity `cap`: value, roofline
    and, with `full`, clocks / e2e / step split / the prefetch-off control."""
    steps = steps or args.steps
    warmup = warmup or args.warmup
    E, N, H, F = s.num_experts, s.tokens, s.hidden, s.ffn
    pool = cap < E
    st = Stack(args, s, dev, rank, world, cap, "host_master" if pool else "device_all",
               weights=weights)
    pf_mb = args.prefetch_mb if args.prefetch_mb >= 0 else (32.0 if not pool else 0.0)
    if pf_mb > 0 and not pool:
        st.set_prefetch(pf_mb)
    h2d_pf = args.h2d_prefetch if h2d_prefetch is None else h2d_prefetch
    if pool and h2d_pf > 0:
        st.set_h2d_prefetch(h2d_pf)
    for i in range(warmup):
        st.step(i)
    torch.cuda.synchronize()
    graphs = not args.eager and not pool
    if graphs:
        st.capture(warmup)
    clk = Clocks(dev.index) if full else None
    ms, _ = st.timed(steps, warmup)
    clocks = clk.stop() if clk else None
    ms_ph, phases = st.timed(steps, warmup, phase_timing=True)
    tot, launches = phase_sums(phases)
    layer_steps = steps * s.layers
    value = N * layer_steps * world / (ms / 1e3)
    res = {"value": round(value, 1), "unit": UNIT, "ms_per_step": round(ms / steps, 4),
           "us_per_layer_step": round(1e3 * ms / layer_steps, 2),
           "workload": workload_str(s, cap, args.interval),
           "launch": "CUDA graph per block step (all layers), replayed" if graphs
                     else "eager stream (PDL-chained kernels)",
           "prefetch_mb": pf_mb, "h2d_prefetch_experts": h2d_pf if pool else 0,
           "gpu_launches": launches, "steps": steps, "warmup": warmup,
           "phases_us_per_layer_step": {kk: round(1e3 * v / layer_steps, 2) for kk, v in tot.items()},
           "ms_per_step_with_phase_events": round(ms_ph / steps, 4)}
    if full:
        res["clocks"] = clocks
        res["step_split"] = st.step_split(steps, warmup)
    acc = st.stats_replay(steps, warmup)
    pk = peaks()
    peak = pk.get("hbm_gbs", 6650.0)
    peak_src = ("measured (MEASURED_PEAKS.json hbm_gbs, device copy)" if "hbm_gbs" in pk
                else "fallback 6.65 TB/s (B200_PROFILING.md)")
    ffn_s = (tot["ffn_ms"] / 1e3) / layer_steps  # the first (resident) FFN launch of a step
    if not pool:
        per_launch = acc["alg"] / layer_steps
        achieved = per_launch / ffn_s / 1e9
        tkey = f"{s.name}|{args.routing}|C={cap}|ep=none|L={s.layers}"
        traffic, tdet = traffic_for(tkey)
        flops = 2 * N * s.top_k * 3 * H * F + (2 * N * 3 * H * F if s.shared_expert else 0)
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "frac_of_nominal_8TBps": round(achieved / 8000.0, 4),
                "kernel": "tide_ffn_kernel (grouped SwiGLU, tcgen05 + TMA)",
                "peak_source": peak_src, "bytes_per_launch": round(per_launch),
                "avg_launch_us": round(ffn_s * 1e6, 2),
                "ffn_share_of_step": round(tot["ffn_ms"] / max(tot["total_ms"], 1e-9), 4),
                "tensor_frac": round(flops / ffn_s / 1e12 / pk.get("bf16_tflops", 1590.0), 5),
                "unique_experts_per_layer_step": round(acc["uniq"] / layer_steps, 2),
                "traffic_key": tkey, "traffic_detail": tdet,
                "l2_prefetch": (f"{pf_mb:g} MB of this layer's likely experts were prefetched "
                                "into L2 by the previous layer's FFN tail and the next "
                                f"{pf_mb / 2:g} MB by this FFN's CTAs before their wait on the "
                                "routing (see frac_prefetch_off)" if pf_mb > 0 else "off")}
        if full and pf_mb > 0:  # control: the same launches with the cross-layer prefetch off
            st.set_prefetch(0)
            _, ph0 = st.timed(steps, warmup, phase_timing=True)
            t0, _ = phase_sums(ph0)
            f0 = (t0["ffn_ms"] / 1e3) / layer_steps
            roof["frac_prefetch_off"] = round(per_launch / f0 / 1e9 / peak, 4)
            roof["avg_launch_us_prefetch_off"] = round(f0 * 1e6, 2)
            st.set_prefetch(pf_mb)
        res["roofline"] = roof
    else:
        pkh = h2d_peak_gbs(dev)
        eff = (acc["h2d"] / steps) / (ms / steps / 1e3) / 1e9
        res_launch = acc["res_alg"] / layer_steps
        res["roofline"] = {
            "bound": "pcie", "achieved": round(eff, 2), "peak": round(pkh, 2), "unit": "GB/s",
            "frac": round(eff / pkh, 4), "traffic": None,
            "kernel": "expert H2D copies (a6, cudaMemcpyAsync on the side stream)",
            "peak_source": "best pinned-host -> HBM copy of 256 MB measured in this run",
            "note": "capacity-limited steps are bound by the H2D link (SURVEY 8(d)): achieved = "
                    "expert bytes copied H2D per step / device time per step",
            "copies_per_step": round(acc["copies"] / steps, 2),
            "h2d_bytes_per_step": round(acc["h2d"] / steps),
            "ffn_resident_launch": {
                "bytes_per_launch": round(res_launch),
                "avg_launch_us": round(ffn_s * 1e6, 2),
                "achieved_gbs": round(res_launch / ffn_s / 1e9, 1),
                "frac_of_hbm_peak": round(res_launch / ffn_s / 1e9 / peak, 4),
                "note": "the step's first FFN launch (experts in HBM at step start + shared) "
                        "timed alone by events on its stream; the staged-chunk launches wait on "
                        "their copies and are not in it"},
            "ffn_launches_per_layer_step": round(acc["launches"] / layer_steps, 2)}
    if full and not args.no_e2e:
        res["e2e"] = st.e2e(steps, warmup, graphs)
    if full and not pool:
        res["routing_stats"] = st.routing_stats()
    st.close()
    del st
    torch.cuda.empty_cache()
    return res


def sub_results(args, dev):
    """N=1 companions of the headline, each a full pass of the hot path measured the same
    way (graphs when every expert is in HBM): BJ.configs[4] the 8-block sweep batch at C = E
    (the mini stack's weights, 256 tokens per layer-step), and BJ.configs[2] the flash-shaped
    stack with pinned-host serving at the paper's budget C = 64 and at C = 217 (8 of its 32
    layers: 206 GB of experts do not fit one GPU)."""
    from paper_2605_20179_b200 import tide
    out = {}
    steps, warmup = min(args.steps, 20), max(3, min(args.warmup, 5))
    try:
        sw = shape_for("sweep")
        desc = tide.make_desc(sw.num_experts, sw.top_k, sw.hidden, sw.ffn, sw.tokens,
                              tide.TIDE_BF16, shared_expert=True)
        w = [gen_layer(args, sw, l, dev, desc) for l in range(sw.layers)]
        out["sweep_8blocks_C256"] = measure_single(args, sw, 256, dev, weights=w, full=False,
                                                   steps=steps, warmup=warmup)
        del w
    except Exception as e:  # reported, not hidden
        out["sweep_8blocks_C256"] = {"error": repr(e)[:300]}
    torch.cuda.empty_cache()
    try:
        fs = shape_for("flash1")
        desc = tide.make_desc(fs.num_experts, fs.top_k, fs.hidden, fs.ffn, fs.tokens,
                              tide.TIDE_BF16)
        w = [gen_layer(args, fs, l, dev, desc, host=True) for l in range(fs.layers)]
        for cap in (64, 217):
            for pf in (0, 8):  # NEXT-3 H2D prefetch off / on (8 experts per layer)
                out[f"flash_C{cap}_8layers" + ("_h2d_prefetch" if pf else "")] = measure_single(
                    args, fs, cap, dev, weights=w, full=False, steps=max(3, steps // 2),
                    warmup=warmup, h2d_prefetch=pf)
        del w
    except Exception as e:
        out["flash_pinned_host"] = {"error": repr(e)[:300]}
    torch.cuda.empty_cache()
    return out


# ------------------------------------------------------------------ expert parallel
def ep_pair_counts(st: Stack, steps, warmup):
    """[P] number of this rank's (token, slot) pairs routed to each rank's experts over the
    timed (layer, t) sequence, for NVLink byte accounting only (an fp32 torch evaluation of
    the router; a near-tie token may land one pair on a different rank than the kernel's)."""
    s = st.s
    cnt = np.zeros(st.world, np.int64)
    for i in range(steps):
        t = (warmup + i) % s.steps
        for L in st.layers:
            lg = L["x"][t].float() @ L["router"].float().T
            top = torch.topk(lg, s.top_k, dim=1).indices
            cnt += np.bincount((top // st.El).flatten().cpu().numpy(), minlength=st.world)
    return cnt


def measure_ep(args, s: g.Shape, dev, rank, world, p2p: bool, weights=None, full=True):
    E, N, H, k = s.num_experts, s.tokens, s.hidden, s.top_k
    El = E // world
    cap = min(args.capacity or El, El)
    st = Stack(args, s, dev, rank, world, cap, "ep", weights=weights, p2p=p2p)
    steps, warmup = args.steps, args.warmup
    pf_mb = args.prefetch_mb if args.prefetch_mb >= 0 else 32.0  # next layer's local experts
    if pf_mb > 0:
        st.set_prefetch(pf_mb)
    for i in range(warmup):
        st.step(i)
    torch.cuda.synchronize()
    graphs = not args.eager
    if graphs:
        try:
            st.capture(warmup)
        except Exception as e:  # capture unsupported in this setting: time eagerly, say so
            st.graphs = None
            graphs = False
            print(f"bench: EP graph capture failed ({e!r}); eager launches", file=sys.stderr)
    clk = Clocks(dev.index) if full else None
    ms, _ = st.timed(steps, warmup)
    clocks = clk.stop() if clk else None
    if p2p:
        errs = [L["ctx"].error() for L in st.layers]
        if any(errs):
            raise RuntimeError(f"peer-memory EP watchdog fired on rank {rank}: {errs}")
    ms_ph, phases = st.timed(steps, warmup, phase_timing=True)
    tot, launches = phase_sums(phases)
    layer_steps = steps * s.layers
    value = N * layer_steps * world / (ms / 1e3)
    check = ep_check(st, args, s, dev, rank, world, p2p) if full else None
    acc = st.stats_replay(steps, warmup)
    pk = peaks()
    peak = pk.get("hbm_gbs", 6650.0)
    ffn_s = (tot["ffn_ms"] / 1e3) / layer_steps
    per_launch = acc["alg"] / layer_steps
    ach = per_launch / ffn_s / 1e9
    ach_min = reduce_over_ranks(ach, world, dev, op="min")
    # NVLink bytes out of / into this rank per layer-step (SURVEY 8(d) metric 5)
    cnt = ep_pair_counts(st, steps, warmup)
    allc = gather_over_ranks(cnt.tolist(), world, dev)  # allc[src][dst] pairs
    peers = world - 1
    y_out = sum(allc[src][rank] for src in range(world) if src != rank) * H * 4 / layer_steps
    y_in = sum(cnt[d] for d in range(world) if d != rank) * H * 4 / layer_steps
    if p2p:
        # router: X rows to every peer + each remote pair's list append at its owner (a 4-byte
        # atomic and two 4-byte stores); FFN epilogue: y rows back to their token's rank
        app_out = sum(cnt[d] for d in range(world) if d != rank) * 12 / layer_steps
        app_in = sum(allc[src][rank] for src in range(world) if src != rank) * 12 / layer_steps
        disp = peers * (N * H * 2 + 4)
        out_b = disp + app_out + y_out + peers * El * 4
        in_b = disp + app_in + y_in + peers * El * 4
        how = ("kernel peer stores: X rows to every peer and each pair's list append at its "
               "expert's owner (router), pair y rows to their token's rank (FFN epilogue), "
               "local counts to every peer")
    else:
        out_b = in_b = peers * (N * (H * 2 + k * 8) + N * H * 4 + El * 4)
        how = ("NCCL: all-gather of [x | top-k | gates] (max_tokens rows per rank), all-to-all "
               "of fp32 partial sums (max_tokens rows per peer), all-gather of local counts")
    lstep_s = ms / 1e3 / layer_steps
    nv = {"bytes_out_per_layer_step": round(out_b), "bytes_in_per_layer_step": round(in_b),
          "gbs_out": round(out_b / lstep_s / 1e9, 2), "peak_gbs": NVLINK_GBS,
          "frac": round(out_b / lstep_s / 1e9 / NVLINK_GBS, 5), "how": how,
          "note": "the rank's NVLink bytes per layer-step / layer-step time: an average over the "
                  "step (a few MB per step are latency-bound, not a link-saturation test)"}
    res = {"value": round(value, 1), "unit": UNIT, "ms_per_step": round(ms / steps, 4),
           "us_per_layer_step": round(1e3 * ms / layer_steps, 2),
           "workload": workload_str(s, cap, args.interval, ep_world=world),
           "exchange": "peer memory (dispatch in the router, combine in the FFN epilogue)" if p2p
                       else "NCCL collectives",
           "launch": "CUDA graph per block step (all layers), replayed" if graphs
                     else "eager stream",
           "prefetch_mb": pf_mb,
           "gpu_launches": launches,
           "roofline": {"bound": "hbm", "achieved": round(ach_min, 1), "peak": peak,
                        "unit": "GB/s", "frac": round(ach_min / peak, 4), "traffic": None,
                        "kernel": "tide_ffn_kernel over the rank's local experts",
                        "rank0_achieved": round(ach, 1) if rank == 0 else None,
                        "note": "min over ranks of the FFN's algorithmic bytes per launch / its "
                                "launch time",
                        "bytes_per_launch": round(per_launch),
                        "avg_launch_us": round(ffn_s * 1e6, 2)},
           "nvlink": nv,
           "phases_us_per_layer_step": {kk: round(1e3 * v / layer_steps, 2) for kk, v in tot.items()}}
    if full:
        res["clocks"] = clocks
        res["ep_check"] = check
        res["step_split"] = st.step_split(steps, warmup)
        if not args.no_e2e:
            res["e2e"] = st.e2e(steps, warmup, graphs)
    w = st.weights()
    st.close()
    del st
    torch.cuda.empty_cache()
    return res, w


# ------------------------------------------------------------------ arms
def run_tide(args, rank: int, world: int, local_rank: int, nccl_ok: bool = True):
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    ep = (args.ep or world > 1) and not args.replicas
    name = args.config or ("flash" if ep and world > 1 else "mini")
    s = shape_for(name, args.layers)
    strong = bool(args.strong and ep)
    if strong:  # 8 blocks in total per layer-step, split over the ranks
        s = g.Shape(s.name, s.num_experts, s.top_k, s.hidden, s.ffn, s.layers,
                    max(1, 8 * 32 // world), s.steps, s.interval, s.capacity, s.dtype,
                    s.shared_expert)
    base = {"metric": METRIC, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True,
            "scaling": "strong" if strong else "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic: tidegen seeded weights (U(+-sqrt(3/fan_in)), bf16) and " +
                    ("calibrated temporal block routing (alpha=0.99, skew=0.5, a0=0.8)"
                     if args.routing == "calibrated" else
                     "uniform iid stress routing (alpha=0, a0=0, skew=0)"),
            "paper_context": PAPER_CONTEXT}
    if ep:
        E = s.num_experts
        p2p = not args.nccl and (world > 1 or args.p2p)
        try:
            head, w = measure_ep(args, s, dev, rank, world, p2p)
        except Exception as e:
            if not p2p or not nccl_ok:
                raise
            print(f"bench: peer-memory EP failed on rank {rank} ({e!r}); NCCL EP is the "
                  f"headline", file=sys.stderr)
            head, w = measure_ep(args, s, dev, rank, world, False)
            head["p2p_error"] = repr(e)[:300]
            p2p = False
        sub = {}
        if p2p and nccl_ok and not args.no_sub:  # the NCCL variant on the same weights
            try:
                sub["nccl_ep"], _ = measure_ep(args, s, dev, rank, world, False, weights=w,
                                               full=False)
            except Exception as e:
                sub["nccl_ep"] = {"error": repr(e)[:300]}
        del w
        res = dict(base, value=head.pop("value"), ms_per_step=head.pop("ms_per_step"),
                   config={"workload": head.pop("workload"), "layers": s.layers,
                           "tokens_per_layer_step_per_rank": s.tokens, "num_experts": E,
                           "top_k": s.top_k, "hidden": s.hidden, "ffn": s.ffn,
                           "capacity_per_rank": min(args.capacity or E // world, E // world),
                           "interval": args.interval, "routing": args.routing,
                           "parallelism": f"expert parallel x{world} (E/P = {E // world} experts "
                                          f"per rank), {head.pop('exchange')}",
                           "l2": "inputs larger than L2: each layer's local weights rotate "
                                 "through the stack between reuses",
                           "launch": head.pop("launch")},
                   roofline=head.pop("roofline"), nvlink=head.pop("nvlink"),
                   e2e=head.pop("e2e", None), clocks=head.pop("clocks", None),
                   gpu_launches=int(head.pop("gpu_launches")) * world,
                   cpu_baseline=None, sub_results=sub)
        res.update(head)
        if world == 1 and rank == 0 and not args.no_cpu:
            res["cpu_baseline"] = cpu_baseline(s, args.seed, args.cpu_seconds, min(s.tokens, 32),
                                               args.routing)
        return res

    cap = args.capacity or s.num_experts
    head = measure_single(args, s, cap, dev, rank, world)
    head.pop("steps"), head.pop("warmup")
    res = dict(base, value=head.pop("value"), ms_per_step=head.pop("ms_per_step"),
               config={"workload": head.pop("workload"), "layers": s.layers,
                       "tokens_per_layer_step": s.tokens, "num_experts": s.num_experts,
                       "top_k": s.top_k, "hidden": s.hidden, "ffn": s.ffn, "capacity": cap,
                       "interval": args.interval, "routing": args.routing,
                       "parallelism": f"replicas x{world} (each rank its own blocks)",
                       "l2": "inputs larger than L2: each layer's weights (>=1.6 GB) rotate "
                             "through the stack between reuses",
                       "launch": head.pop("launch"), "prefetch_mb": head.pop("prefetch_mb")},
               roofline=head.pop("roofline"), e2e=head.pop("e2e", None),
               clocks=head.pop("clocks", None),
               gpu_launches=int(head.pop("gpu_launches")) * world, cpu_baseline=None)
    res.update(head)
    if world == 1 and rank == 0 and not args.no_cpu:  # the CPU baseline is an N=1 figure
        res["cpu_baseline"] = cpu_baseline(s, args.seed, args.cpu_seconds, min(s.tokens, 32),
                                           args.routing)
    if (world == 1 and not args.no_sub and args.config is None and not args.layers
            and not args.capacity and args.routing == "calibrated"):
        res["sub_results"] = sub_results(args, dev)
    return res


def run_reference(args, world: int):
    """Reference arm of this tier: the fp64 CPU oracle, as it stands, timed on every host core
    (OpenMP over tokens) on the bench workload's layer-steps (layer 0 of the stack, the
    block's full token count)."""
    import oracle
    ep = (args.ep or world > 1) and not args.replicas
    s = shape_for(args.config or ("flash" if ep and world > 1 else "mini"), args.layers)
    N = s.tokens
    uni = args.routing == "uniform"
    wr, wg, wu, wd, sh = g.layer_torch(s, args.seed, 0, "cpu", skew=0.0 if uni else g.SKEW)
    to = g.torch_to_np
    L = oracle.Layer(to(wr), to(wg), to(wu), to(wd), tuple(to(a) for a in sh) if sh else None)
    del wg, wu, wd
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
              f"OpenMP over tokens) of layer 0 of the stack on all {N} tokens of one block")
    return {"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * el / args.steps, 2), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_str(s, cap, args.interval), "layers": s.layers,
                       "tokens_per_layer_step": s.tokens, "num_experts": E, "top_k": s.top_k,
                       "hidden": s.hidden, "ffn": s.ffn, "capacity": cap,
                       "interval": args.interval, "routing": args.routing,
                       "oracle_sample": f"layer 0 of {s.layers}, all {N} tokens per step, on "
                                        f"rank 0 (the oracle has no multi-GPU form)"},
            "cpu_baseline": {"value": round(v, 3), "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": sample, "host_cpu": _cpu_model()},
            "e2e": {"value": round(v, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


_OUT = sys.stdout


def _free_port() -> int:
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    p = so.getsockname()[1]
    so.close()
    return p


def spawn(args) -> int:
    """`python bench.py --gpus N` without torchrun: launch N ranks through torchrun on this
    node (one process per GPU); fails loudly when the node has fewer GPUs."""
    n = torch.cuda.device_count()
    if n < args.gpus and not os.environ.get("TIDE_BENCH_SAME_DEVICE"):
        print(f"bench.py: --gpus {args.gpus} but this node has {n} CUDA device(s)", file=sys.stderr)
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port",
           str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, stdout=_OUT)


def main():
    args = parse()
    # stdout carries the one JSON line: anything native code prints (NCCL's version banner,
    # init lines) goes to stderr, the line itself to the saved stdout
    sys.stdout.flush()
    out_fd = os.dup(1)
    os.dup2(2, 1)
    global _OUT
    _OUT = os.fdopen(out_fd, "w")
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is None and args.gpus > 1:
        sys.exit(spawn(args))
    world = int(world_env or "1")
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":  # the oracle has no multi-GPU form: rank 0 alone
        if rank == 0:
            print(json.dumps(run_reference(args, world)), file=_OUT, flush=True)
        return
    # test mode for the multi-process code path on a one-GPU box: every rank on cuda:0 and a
    # gloo process group (NCCL refuses two ranks per device); replicas and peer-memory EP only
    same_dev = bool(os.environ.get("TIDE_BENCH_SAME_DEVICE"))
    if same_dev:
        local_rank = 0
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # stdout carries the JSON line only
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # keep the NCCL init lines (comm size)
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        torch.cuda.set_device(local_rank)
        if same_dev:
            torch.distributed.init_process_group("gloo")
        else:
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    res = run_tide(args, rank, world, local_rank, nccl_ok=not (same_dev and world > 1))
    if rank == 0:
        print(json.dumps(res), file=_OUT, flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
