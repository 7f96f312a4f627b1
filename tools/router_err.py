"""Max |GPU logit - fp64 oracle logit| of the router for the bench shapes (R-17 budget 6e-7).
usage: python tools/router_err.py   (TIDE_ROUTER_CC=1: CUDA-core kernel)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import tidegen as g  # noqa: E402
from paper_2605_20179_b200 import tide  # noqa: E402

for name, tokens in (("mini", 32), ("flash", 32), ("sweep", 256)):
    shape = g.SHAPES[name]
    E, H = shape.num_experts, shape.hidden
    worst = 0.0
    for seed in (51, 52, 53):
        wr = g.router_np(shape, seed, 0)
        x = g.block_hidden_np(shape, seed, steps=1, tokens=tokens)[0]
        ref = oracle.router_logits(x, wr)
        desc = tide.make_desc(E, shape.top_k, H, 64, tokens)
        ctx = tide.Context(desc, E)
        dev_all = torch.zeros(E, 3 * H * 64, dtype=torch.bfloat16, device="cuda")
        r = ctx.moe_step(g.np_to_torch(x, "cuda"), g.np_to_torch(wr, "cuda"), device_all=dev_all,
                         placement=torch.zeros(E, dtype=torch.uint8, device="cuda"), step=0,
                         interval=1, debug=True)
        torch.cuda.synchronize()
        worst = max(worst, float(np.abs(r.debug["logits"].cpu().numpy().astype(np.float64) - ref).max()))
    print(f"{name:6s} N={tokens:4d}  max |logit err| = {worst:.3e}")
