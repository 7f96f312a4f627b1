"""Per-item timeline of the FFN kernel (debug ffn_item_trace) on a mini layer: where does a
launch spend the time that the byte stream does not explain?
usage: python tools/ffn_items.py [mini|sweep|flash] [step] [uniform]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tidegen as g  # noqa: E402
from paper_2605_20179_b200 import tide  # noqa: E402

shape = g.SHAPES[sys.argv[1] if len(sys.argv) > 1 else "mini"]
T_AT = int(sys.argv[2]) if len(sys.argv) > 2 else 12
uni = len(sys.argv) > 3 and sys.argv[3] == "uniform"
dev = "cuda"
E, k, H, F, N = shape.num_experts, shape.top_k, shape.hidden, shape.ffn, shape.tokens
desc = tide.make_desc(E, k, H, F, N, shared_expert=shape.shared_expert)
layers = []
for l in range(4):  # rotate 4 layers so the traced layer's weights are cold in L2
    wr, wg, wu, wd, sh = g.layer_torch(shape, 7, l, dev, skew=0.0 if uni else g.SKEW)
    layers.append((wr, tide.pack_layer(desc, wg, wu, wd),
                   torch.cat([a.reshape(-1) for a in sh]) if sh else None,
                   tide.Context(desc, E), g.block_hidden_torch(shape, 7, l, dev, iid=uni)))
    del wg, wu, wd
pl = torch.zeros(E, dtype=torch.uint8, device=dev)
for t in range(T_AT + 1):
    for li, (wr, packed, shared, ctx, xs) in enumerate(layers):
        rr = ctx.moe_step(xs[t], wr, device_all=packed, shared_w=shared, placement=pl, step=t,
                          interval=4, debug=("trace" if (li == 0 and t == T_AT) else False))
        if li == 0 and t == T_AT:
            r = rr
torch.cuda.synchronize()
nsm = torch.cuda.get_device_properties(0).multi_processor_count
ct = r.debug["ffn_trace"].cpu().numpy().reshape(nsm, 8).astype(np.int64)
it = r.debug["ffn_item_trace"].cpu().numpy().reshape(nsm, 64, 4).astype(np.int64)
t0 = ct[:, 0].min()
us = lambda v: (v - t0) / 1e3  # noqa: E731
print(f"{shape.name} t={T_AT} {'uniform' if uni else 'calibrated'}: CTA entry spread "
      f"{us(ct[:, 0].max()):.2f}  list ready {us(ct[:, 1].min()):.2f}..{us(ct[:, 1].max()):.2f}  "
      f"producer done med {us(np.median(ct[:, 2])):.2f} max {us(ct[:, 2].max()):.2f}  "
      f"epilogue done med {us(np.median(ct[:, 3])):.2f} max {us(ct[:, 3].max()):.2f}")
kinds = {0: [], 1: []}
dep, dur, gaps = [], {0: [], 1: []}, []
first_claim = []
for c in range(nsm):
    n = int(ct[c, 4])
    rows = it[c, :min(n, 64)]
    if len(rows) == 0:
        continue
    first_claim.append(us(rows[0, 0]))
    for i, (tc, meta, td, ti) in enumerate(rows):
        kind = int(meta) >> 32
        if kind == 1:
            dep.append((td - tc) / 1e3)
        nxt = rows[i + 1, 0] if i + 1 < len(rows) else ct[c, 2]
        dur[kind].append((nxt - tc) / 1e3)
dep = np.array(dep)
print(f"  items/CTA {ct[:, 4].mean():.1f}; first claim {min(first_claim):.2f}..{max(first_claim):.2f} us")
for kd in (0, 1):
    d = np.array(dur[kd])
    if len(d):
        print(f"  phase-{kd + 1} items {len(d):5d}: claim-to-next-claim med {np.median(d):6.2f} "
              f"p90 {np.percentile(d, 90):6.2f} max {d.max():6.2f} us")
if len(dep):
    print(f"  phase-2 dependency wait: total {dep.sum():8.2f} CTA-us, items waiting > 0.5 us: "
          f"{(dep > 0.5).sum()} of {len(dep)}, max {dep.max():.2f} us")
# utilisation over time: number of CTAs between their first claim and producer done
grid = np.arange(0, us(ct[:, 3].max()) + 1, 1.0)
busy = [(np.array(first_claim) <= x).sum() - (us(ct[:, 2]) < x).sum() for x in grid]
print("  CTAs issuing (per 4 us):", " ".join(str(int(b)) for b in busy[::4]))
# aggregate weight-stream rate over time: each item's bytes spread evenly over claim -> next
# claim of its CTA (phase 1: gate + up tiles, 2 x 128 rows x H; phase 2: 128 down rows x F)
eb = 2 if shape.dtype == "bf16" else 4
b_item = {0: 2 * 128 * H * eb, 1: 128 * F * eb}
bins = np.zeros(int(us(ct[:, 3].max())) + 2)
tot = 0.0
for c in range(nsm):
    n = int(ct[c, 4])
    rows = it[c, :min(n, 64)]
    for i, (tc, meta, td, ti) in enumerate(rows):
        kind = int(meta) >> 32
        nxt = rows[i + 1, 0] if i + 1 < len(rows) else ct[c, 2]
        a, b = us(tc), us(nxt)
        if b <= a:
            continue
        tot += b_item[kind]
        rate = b_item[kind] / (b - a)
        for x in range(int(a), int(b) + 1):
            lo, hi = max(a, x), min(b, x + 1)
            if hi > lo:
                bins[x] += rate * (hi - lo)
print(f"  weight bytes traced {tot / 1e6:.1f} MB; stream rate per 2 us (TB/s):")
print("   ", " ".join(f"{(bins[i] + bins[i + 1]) / 2e6:.2f}" for i in range(0, len(bins) - 1, 2)))
