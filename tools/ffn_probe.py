"""FFN streaming rate vs routing shape: calibrated vs uniform routing at several token counts.
Per case: 4 mini layers rotating (weights >> L2), T steps, per-phase CUDA events
(tide_ctx_set_timing); prints FFN us per launch, unique experts U, algorithmic bytes, TB/s.
usage: python tools/ffn_probe.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tidegen as g  # noqa: E402
from paper_2605_20179_b200 import tide  # noqa: E402

dev = "cuda"
base = g.MINI
E, k, H, F = base.num_experts, base.top_k, base.hidden, base.ffn
NL, T = 4, 16
cache = {}


def weights(skew):
    if skew not in cache:
        ws = []
        for l in range(NL):
            wr, wg, wu, wd, sh = g.layer_torch(base, 7, l, dev, skew=skew)
            d = tide.make_desc(E, k, H, F, 256, shared_expert=True)
            ws.append((wr, tide.pack_layer(d, wg, wu, wd), torch.cat([a.reshape(-1) for a in sh])))
            del wg, wu, wd
        cache[skew] = ws
    return cache[skew]


for routing, N in (("calibrated", 32), ("uniform", 32), ("uniform", 16), ("uniform", 8),
                   ("calibrated", 64), ("calibrated", 16)):
    uni = routing == "uniform"
    ws = weights(0.0 if uni else g.SKEW)
    desc = tide.make_desc(E, k, H, F, N, shared_expert=True)
    shape = g.Shape("p", E, k, H, F, NL, N, steps=T, shared_expert=True)
    ctxs = [tide.Context(desc, E) for _ in range(NL)]
    xs = [g.block_hidden_torch(shape, 7, l, dev, iid=uni) for l in range(NL)]
    pls = [torch.zeros(E, dtype=torch.uint8, device=dev) for _ in range(NL)]
    for rep in range(2):  # rep 0 warm-up, rep 1 timed
        for c in ctxs:
            c.set_timing(rep == 1)
        U = 0
        for t in range(T):
            for l in range(NL):
                r = ctxs[l].moe_step(xs[l][t], ws[l][0], device_all=ws[l][1], shared_w=ws[l][2],
                                     placement=pls[l], step=t, interval=4, placement_out=pls[l],
                                     stats=(rep == 1))
                if rep == 1:
                    U += r.stats["unique_experts"] + 1
        torch.cuda.synchronize()
    ph = [c.timing() for c in ctxs]
    n = T * NL
    ffn_us = sum(p["ffn_ms"] for p in ph) / n * 1e3
    R = N * k + N
    byts = U / n * 3 * H * F * 2 + R * (2 * H + 4 * F + 4 * H)
    print(f"{routing:10s} N={N:3d}: U={U / n:6.1f}  FFN {ffn_us:7.2f} us  {byts / 1e6:7.1f} MB  "
          f"{byts / ffn_us / 1e6:6.3f} TB/s  (route {sum(p['router_ms'] for p in ph) / n * 1e3:5.2f} us)",
          flush=True)
