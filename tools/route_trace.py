"""Trace the fused route kernel's phases with %globaltimer (debug struct route_trace).
usage: python tools/route_trace.py [mini|sweep]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tidegen as g  # noqa: E402
from paper_2605_20179_b200 import tide  # noqa: E402

shape = g.SHAPES[sys.argv[1] if len(sys.argv) > 1 else "mini"]
dev = "cuda"
E, k, H, F, N = shape.num_experts, shape.top_k, shape.hidden, shape.ffn, shape.tokens
desc = tide.make_desc(E, k, H, F, N, shared_expert=shape.shared_expert)
wr, wg, wu, wd, sh = g.layer_torch(shape, 7, 0, dev)
packed = tide.pack_layer(desc, wg, wu, wd)
shared = torch.cat([a.reshape(-1) for a in sh]) if sh else None
ctx = tide.Context(desc, E)
xs = g.block_hidden_torch(shape, 7, 0, dev)
pl = torch.zeros(E, dtype=torch.uint8, device=dev)
for t in range(8):
    r = ctx.moe_step(xs[t], wr, device_all=packed, shared_w=shared, placement=pl, step=t,
                     interval=4, debug=True)
torch.cuda.synchronize()
tr = r.debug["route_trace"].cpu().numpy().reshape(-1, 8).astype(np.int64)
tpc = 4 if N <= 64 else 8
ny = max(1, (N + tpc - 1) // tpc)
tr = tr[tr[:, 0] > 0]  # the CTAs the launched grid had (CUDA-core or tensor-core router)
t0 = tr[:, 0].min()
print(f"{shape.name}: {len(tr)} CTAs")
print(f"  start spread       {(tr[:, 0].max() - t0) / 1e3:7.2f} us")
print(f"  phase1 end (max)   {(tr[:, 1].max() - t0) / 1e3:7.2f} us   median {(np.median(tr[:, 1]) - t0) / 1e3:7.2f}")
last = tr[tr[:, 2] > 0]
print(f"  phase2 CTAs        {len(last)}")
print(f"  phase2 start (min/max) {(last[:, 2].min() - t0) / 1e3:7.2f} / {(last[:, 2].max() - t0) / 1e3:7.2f} us")
print(f"  phase2 end   (max)     {(last[:, 3].max() - t0) / 1e3:7.2f} us")
print(f"  phase2 duration median {np.median(last[:, 3] - last[:, 2]) / 1e3:7.2f} us")
for i, name in ((4, "logits in"), (5, "selection done"), (6, "histogram done")):
    v = last[last[:, i] > 0]
    if len(v):
        print(f"  phase2 {name:15s} median {np.median(v[:, i] - v[:, 2]) / 1e3:7.2f} us after its start")
