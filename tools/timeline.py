"""Timeline of consecutive layer-steps from the kernels' own %globaltimer traces
(route_trace, ffn_trace): where the ~108 us of a mini layer-step go.
usage: python tools/timeline.py [mini|sweep|flash] [t]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tidegen as g  # noqa: E402
from paper_2605_20179_b200 import tide  # noqa: E402

shape = g.SHAPES[sys.argv[1] if len(sys.argv) > 1 else "mini"]
T_AT = int(sys.argv[2]) if len(sys.argv) > 2 else 16
dev = "cuda"
E, k, H, F, N = shape.num_experts, shape.top_k, shape.hidden, shape.ffn, shape.tokens
desc = tide.make_desc(E, k, H, F, N, shared_expert=shape.shared_expert)
NL = 6
layers = []
for l in range(NL):
    wr, wg, wu, wd, sh = g.layer_torch(shape, 7, l, dev)
    layers.append(dict(wr=wr, w=tide.pack_layer(desc, wg, wu, wd),
                       sh=torch.cat([a.reshape(-1) for a in sh]) if sh else None,
                       ctx=tide.Context(desc, E), x=g.block_hidden_torch(shape, 7, l, dev),
                       pl=torch.zeros(E, dtype=torch.uint8, device=dev)))
    del wg, wu, wd
res = []
for t in range(T_AT + 1):
    res = []
    for L in layers:
        res.append(L["ctx"].moe_step(L["x"][t], L["wr"], device_all=L["w"], shared_w=L["sh"],
                                     placement=L["pl"], step=t, interval=4, placement_out=L["pl"],
                                     debug=("trace" if t == T_AT else False)))
torch.cuda.synchronize()
tpc = int(os.environ.get("TIDE_ROUTE_TPC", 4 if N <= 64 else 8))
ny = max(1, (N + tpc - 1) // tpc)
rows = []
for li, r in enumerate(res):
    rt = r.debug["route_trace"].cpu().numpy().reshape(-1, 8).astype(np.int64)
    rt = rt[rt[:, 0] > 0]
    ft = r.debug["ffn_trace"].cpu().numpy().reshape(-1, 8).astype(np.int64)
    ft = ft[ft[:, 0] > 0]
    last = rt[rt[:, 2] > 0]
    rows.append(dict(r0=rt[:, 0].min(), r1=rt[:, 1].max(), r2s=last[:, 2].min(), r2=last[:, 3].max(),
                     f0=ft[:, 0].min(), fl=ft[:, 1].min(), flx=ft[:, 1].max(), fp=ft[:, 2].max(),
                     fe=ft[:, 3].max(), fe_med=np.median(ft[:, 3]), fw=ft[:, 5].min(),
                     fwx=ft[:, 5].max(), r0x=rt[:, 0].max(), c0=ft[0, 6], c1=ft[0, 7],
                     p1med=np.median(rt[:, 1] - rt[:, 0]), p2med=np.median(last[:, 3] - last[:, 2]),
                     p2_load=np.median(last[:, 4] - last[:, 2]), p2_sel=np.median(last[:, 5] - last[:, 4]),
                     p2_atom=np.median(last[:, 6] - last[:, 5]), p2_sync=np.median(last[:, 3] - last[:, 6])))
t0 = rows[1]["r0"]
us = lambda v: (v - t0) / 1e3  # noqa: E731
print(f"{shape.name} t={T_AT}: times in us relative to layer 1's route start")
for li in range(1, NL):
    R = rows[li]
    print(f" layer {li}: route {us(R['r0']):7.2f} .. p1 end {us(R['r1']):7.2f} .. p2 {us(R['r2s']):7.2f}-{us(R['r2']):7.2f} | "
          f"ffn entry {us(R['f0']):7.2f} pdl-wait done {us(R['fw']):7.2f}/{us(R['fwx']):7.2f} list {us(R['fl']):7.2f}/{us(R['flx']):7.2f} prod-done {us(R['fp']):7.2f} "
          f"epi med {us(R['fe_med']):7.2f} max {us(R['fe']):7.2f}")
    print(f"   combine start (latest) {us(R['c0']):7.2f} end (latest) {us(R['c1']):7.2f}")
    print(f"   route CTA start spread {(R['r0x'] - R['r0']) / 1e3:5.2f}  per-CTA phase1 median {R['p1med'] / 1e3:5.2f}"
          f"  phase2 median {R['p2med'] / 1e3:5.2f} = logits {R['p2_load'] / 1e3:5.2f} + select "
          f"{R['p2_sel'] / 1e3:5.2f} + histogram atomics {R['p2_atom'] / 1e3:5.2f} + barrier "
          f"{R['p2_sync'] / 1e3:5.2f}")
    if li + 1 < NL:
        print(f"   gap ffn end -> next route start {us(rows[li + 1]['r0']) - us(R['fe']):6.2f} us "
              f"(combine + launch)")
per = (rows[NL - 1]["r0"] - rows[1]["r0"]) / (NL - 2) / 1e3
print(f" mean layer-step period {per:.2f} us")
