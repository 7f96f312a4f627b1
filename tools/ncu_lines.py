"""Summarise an ncu report's source page per CUDA line: top lines by warp-stall samples.
usage: python tools/ncu_lines.py report.ncu-rep [function-substring] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
filt = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
func, hdr, rows = None, None, {}
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "Function Name":
        func = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or func is None or filt not in func or not r[0].isdigit():
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        s = 0
    key = (func[:60], int(r[0]))
    ent = rows.setdefault(key, [0, r[1][:90], {}])
    ent[0] += s
    for k, v in d.items():
        if k.startswith("stall_"):
            try:
                ent[2][k] = ent[2].get(k, 0) + int(v)
            except ValueError:
                pass
tot = {}
for (f, _), e in rows.items():
    tot[f] = tot.get(f, 0) + e[0]
for f, t in tot.items():
    print(f"== {f}  total samples {t}")
    items = sorted(((e[0], ln, e[1], e[2]) for (ff, ln), e in rows.items() if ff == f), reverse=True)
    for s, ln, src, st in items[:top]:
        worst = sorted(st.items(), key=lambda kv: -kv[1])[:3]
        print(f"{s:7d} {100*s/max(t,1):5.1f}%  L{ln:4d}  {src:90s} {worst}")
