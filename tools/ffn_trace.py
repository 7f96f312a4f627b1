"""Trace the FFN kernel per CTA (debug ffn_trace) on a mini/flash layer at step t.
usage: python tools/ffn_trace.py [mini|sweep|flash] [steps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tidegen as g  # noqa: E402
from paper_2605_20179_b200 import tide  # noqa: E402

shape = g.SHAPES[sys.argv[1] if len(sys.argv) > 1 else "mini"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 12
dev = "cuda"
E, k, H, F, N = shape.num_experts, shape.top_k, shape.hidden, shape.ffn, shape.tokens
desc = tide.make_desc(E, k, H, F, N, shared_expert=shape.shared_expert)
layers = []
for l in range(4):  # rotate 4 layers (>= 6 GB) so the traced layer's weights are cold in L2
    wr, wg, wu, wd, sh = g.layer_torch(shape, 7, l, dev)
    layers.append((wr, tide.pack_layer(desc, wg, wu, wd),
                   torch.cat([a.reshape(-1) for a in sh]) if sh else None,
                   tide.Context(desc, E), g.block_hidden_torch(shape, 7, l, dev)))
    del wg, wu, wd
pl = torch.zeros(E, dtype=torch.uint8, device=dev)
for t in range(steps):
    for li, (wr, packed, shared, ctx, xs) in enumerate(layers):
        rr = ctx.moe_step(xs[t], wr, device_all=packed, shared_w=shared, placement=pl, step=t,
                          interval=4, debug=(li == 0), stats=(li == 0))
        if li == 0:
            r = rr
torch.cuda.synchronize()
tr = r.debug["ffn_trace"].cpu().numpy().reshape(-1, 8).astype(np.int64)
t0 = tr[:, 0].min()
us = lambda v: (v - t0) / 1e3  # noqa: E731
print(f"{shape.name} layer 0 step {steps - 1}: unique experts {r.stats['unique_experts']}, "
      f"weight bytes {r.stats['weight_bytes_read'] / 1e6:.1f} MB")
print(f"  entry spread          {us(tr[:, 0].max()):7.2f} us")
print(f"  work list ready       min {us(tr[:, 1].min()):7.2f}  max {us(tr[:, 1].max()):7.2f}")
print(f"  producer done         min {us(tr[:, 2].min()):7.2f}  med {us(np.median(tr[:, 2])):7.2f}  max {us(tr[:, 2].max()):7.2f}")
print(f"  epilogue done         min {us(tr[:, 3].min()):7.2f}  med {us(np.median(tr[:, 3])):7.2f}  max {us(tr[:, 3].max()):7.2f}")
print(f"  items per CTA         min {tr[:, 4].min()}  max {tr[:, 4].max()}  total {tr[:, 4].sum()}")
busy = us(tr[:, 3].max()) - us(tr[:, 1].min())
print(f"  weight stream {r.stats['weight_bytes_read'] / 1e6:.1f} MB over {busy:.1f} us from list-ready to last epilogue "
      f"= {r.stats['weight_bytes_read'] / busy / 1e6:.2f} TB/s")
