"""DRAM traffic of tide_ffn_kernel vs its algorithmic bytes, launch by launch.

  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --print-units base --clock-control none -k regex:tide_ffn -c <L*T> --csv --log-file gpurun_out/ffn_<cfg>.csv \
      python tools/ffn_traffic.py --config mini --algo gpurun_out/ffn_<cfg>_algo.json
  python tools/ffn_traffic.py --config mini --join gpurun_out/ffn_<cfg>.csv \
      --algo gpurun_out/ffn_<cfg>_algo.json  # -> profiles/ffn_traffic.json["<cfg>|calibrated|C=256|ep=none|L=<layers>"]

The run pushes exactly one block (t = 0..T-1) through the whole stack in bench.py's order
(layer-major within a step, C = E, interval 4). The first L*T FFN launches are the ones
ncu captures. Afterwards the same sequence is replayed with stats (routing is deterministic),
and each launch's algorithmic bytes are written ((U+shared)*3HF*2 + R*(2H+4F+4H)).
"""
import argparse
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="mini")
ap.add_argument("--layers", type=int, default=0)
ap.add_argument("--algo", required=True)
ap.add_argument("--join", default="")
a = ap.parse_args()

if a.join:
    rows = list(csv.reader(open(a.join)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ii, mi, vi = h.index("ID"), h.index("Metric Name"), h.index("Metric Value")
    per = {}
    for r in rows[hi + 1:]:
        if len(r) > vi:
            per.setdefault(int(r[ii]), {})[r[mi]] = float(r[vi].replace(",", ""))
    launches = [per[i] for i in sorted(per)]
    algo = json.load(open(a.algo))
    n = min(len(launches), len(algo["bytes"]))
    dram = [x["dram__bytes_read.sum"] + x["dram__bytes_write.sum"] for x in launches[:n]]
    dur = [x["gpu__time_duration.sum"] for x in launches[:n]]  # ns
    alg = algo["bytes"][:n]
    res = {"dram_bytes_per_launch": round(sum(dram) / n),
           "algorithmic_bytes_per_launch": round(sum(alg) / n),
           "dram_over_algorithmic": round(sum(dram) / sum(alg), 4),
           "launches": n,
           "ncu_serialised_cold_l2_TBps": round(sum(dram) / sum(dur) / 1e3, 3),
           "ncu_algorithmic_TBps": round(sum(alg) / sum(dur) / 1e3, 3),
           "mean_launch_us_ncu": round(sum(dur) / n / 1e3, 2),
           "note": (f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
                    f"gpu__time_duration.sum --clock-control none over every FFN launch of one "
                    f"block ({algo['layers']} layers x T={algo['T']}, t=0..T-1), cold L2 per "
                    f"launch; algorithmic bytes from a stats replay of the same launches "
                    f"(tools/ffn_traffic.py)")}
    out = os.path.join(ROOT, "profiles", "ffn_traffic.json")
    allr = json.load(open(out)) if os.path.exists(out) else {}
    key = f"{a.config}|calibrated|C=256|ep=none|L={algo['layers']}"  # bench.py's lookup key
    res["config"] = {"shape": a.config, "routing": "calibrated", "capacity": 256, "ep": "none",
                     "layers": algo["layers"]}
    allr[key] = res
    json.dump(allr, open(out, "w"), indent=1)
    print(json.dumps(res))
    sys.exit(0)

import torch  # noqa: E402
import tidegen as g  # noqa: E402
from paper_2605_20179_b200 import tide  # noqa: E402

s = {"mini": g.MINI, "sweep": g.SWEEP, "flash1": g.FLASH}[a.config]
Lyr = a.layers or (8 if a.config == "flash1" else s.layers)
E, k, H, F, N, T = s.num_experts, s.top_k, s.hidden, s.ffn, s.tokens, s.steps
dev = torch.device("cuda")
desc = tide.make_desc(E, k, H, F, N, tide.TIDE_BF16, shared_expert=s.shared_expert)
layers = []
for l in range(Lyr):
    wr, wg, wu, wd, sh = g.layer_torch(s, 7, l, dev)
    packed = tide.pack_layer(desc, wg, wu, wd)
    del wg, wu, wd
    shared = torch.cat([t.reshape(-1) for t in sh]) if sh else None
    layers.append(dict(wr=wr, w=packed, sh=shared, ctx=tide.Context(desc, E),
                       x=g.block_hidden_torch(s, 7, l, dev),
                       pl=torch.zeros(E, dtype=torch.uint8, device=dev)))


def run(stats):
    out = []
    for L in layers:
        L["pl"].zero_()
    for t in range(T):
        for L in layers:
            r = L["ctx"].moe_step(L["x"][t], L["wr"], device_all=L["w"], shared_w=L["sh"],
                                  placement=L["pl"], step=t, interval=4, placement_out=L["pl"],
                                  stats=stats)
            if stats:
                u = r.stats["unique_experts"] + (1 if s.shared_expert else 0)
                R = N * k + (N if s.shared_expert else 0)
                out.append(u * s.expert_bytes + R * (H * 2 + 2 * F * 2 + H * 4))
    torch.cuda.synchronize()
    return out


run(False)          # the launches ncu captures (first L*T FFN launches)
alg = run(True)     # same sequence, algorithmic bytes per launch
json.dump({"config": a.config, "layers": Lyr, "T": T, "bytes": alg}, open(a.algo, "w"))
print(f"{len(alg)} launches, mean algorithmic {sum(alg) / len(alg) / 1e6:.1f} MB")
