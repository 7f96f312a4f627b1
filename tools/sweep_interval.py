"""BJ.configs[4]: refresh-interval x capacity sweep on the mini shape with a batch of 8 blocks
(256 tokens per layer-step), pinned-host serving of non-resident experts.

For every (capacity C, interval tau): one full block (T = 32 steps) of layer-steps on
`--layers` layers, timed with CUDA events; H2D copies from the library's stats.  Then the
NEXT-2 model: drift d measured on the GPU (tide_trace_stats, Eq. 4, top-C of each step's
hits), c_io = c_miss = measured seconds per expert H2D copy (a miss streams the expert,
R-13), tau* from tide_optimize_interval, compared with the measured best tau per C.
usage: python tools/sweep_interval.py [--layers 2] [--out profiles/r01/sweep_interval.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tidegen as g  # noqa: E402
from paper_2605_20179_b200 import tide  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=2)
ap.add_argument("--caps", default="64,128,192,256")
ap.add_argument("--taus", default="1,2,4,8,16")
ap.add_argument("--out", default="profiles/r01/sweep_interval.json")
a = ap.parse_args()
s = g.SWEEP
E, k, H, F, N, T = s.num_experts, s.top_k, s.hidden, s.ffn, s.tokens, s.steps
dev = "cuda"
desc = tide.make_desc(E, k, H, F, N, shared_expert=True)
xb = tide.expert_bytes(desc)
layers = []
for l in range(a.layers):
    wr, wg, wu, wd, sh = g.layer_torch(s, 7, l, dev)
    packed = tide.pack_layer(desc, wg, wu, wd)
    del wg, wu, wd
    host = packed.cpu().pin_memory()
    del packed
    torch.cuda.empty_cache()
    layers.append(dict(wr=wr, host=host, shared=torch.cat([t.reshape(-1) for t in sh]),
                       x=g.block_hidden_torch(s, 7, l, dev)))
# measured H2D cost of one expert (pinned -> HBM)
buf = torch.empty(xb // 2, dtype=torch.bfloat16, device=dev)
src = layers[0]["host"][0]
for _ in range(3):
    buf.copy_(src, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(20):
    buf.copy_(layers[0]["host"][i], non_blocking=True)
e1.record()
torch.cuda.synchronize()
c_io = e0.elapsed_time(e1) / 1e3 / 20
print(f"H2D per expert {c_io * 1e6:.1f} us ({xb / c_io / 1e9:.1f} GB/s)", flush=True)

# routing trace of layer 0 over the block (device_all run, interval 1) -> drift per capacity
ctx = tide.Context(desc, E)
dall = layers[0]["host"].to(dev)
counts = torch.empty(T, E, dtype=torch.int32, device=dev)
pl = torch.zeros(E, dtype=torch.uint8, device=dev)
for t in range(T):
    ctx.moe_step(layers[0]["x"][t], layers[0]["wr"], device_all=dall, shared_w=layers[0]["shared"],
                 placement=pl, step=t, interval=1, hit_counts=counts[t])
del dall
torch.cuda.empty_cache()

res = {"workload": "BJ.configs[4]: mini shape, 8 blocks (256 tokens) per layer-step, "
                   f"{a.layers} layers, T={T}, pinned-host serving (host_master)",
       "h2d_us_per_expert": c_io * 1e6, "runs": [], "model": []}
for C in [int(v) for v in a.caps.split(",")]:
    sim, uq, drift = tide.trace_stats(counts, C)
    d = float(drift.mean().item())
    tau_star, curve = tide.optimize_interval(T, C, d, c_io, c_io)
    res["model"].append({"capacity": C, "drift_mean": d, "tau_star": tau_star,
                         "curve_ms": [round(v * 1e3, 3) for v in curve[:16]]})
    for tau in [int(v) for v in a.taus.split(",")]:
        ctxs = [tide.Context(desc, C, 16) for _ in layers]
        pls = [torch.zeros(E, dtype=torch.uint8, device=dev) for _ in layers]
        stats = dict(copies=0, h2d=0, resident_pairs=0, pairs=0)
        torch.cuda.synchronize()
        e0.record()
        for t in range(T):
            for L, c, p in zip(layers, ctxs, pls):
                r = c.moe_step(L["x"][t], L["wr"], host_master=L["host"], shared_w=L["shared"],
                               placement=p, step=t, interval=tau, placement_out=p, stats=True)
                stats["copies"] += r.stats["copies"]
                stats["h2d"] += r.stats["h2d_bytes"]
                stats["resident_pairs"] += r.stats["resident_pairs"]
                stats["pairs"] += N * k
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        ls = T * len(layers)
        row = {"capacity": C, "interval": tau, "ms_per_layer_step": ms / ls,
               "block_tokens_per_s": N * ls / (ms / 1e3),
               "h2d_experts_per_layer_step": stats["copies"] / ls,
               "h2d_GBps": stats["h2d"] / (ms / 1e3) / 1e9,
               "resident_pair_rate": stats["resident_pairs"] / stats["pairs"]}
        res["runs"].append(row)
        print(json.dumps(row), flush=True)
        del ctxs
for C in [int(v) for v in a.caps.split(",")]:
    rows = [r for r in res["runs"] if r["capacity"] == C]
    best = max(rows, key=lambda r: r["block_tokens_per_s"])
    m = [x for x in res["model"] if x["capacity"] == C][0]
    m["measured_best_tau"] = best["interval"]
os.makedirs(os.path.dirname(a.out), exist_ok=True)
json.dump(res, open(a.out, "w"), indent=1)
print(json.dumps(res["model"]))
