"""Key metrics of an `ncu --set full` report as JSON (one entry per profiled launch).
usage: python tools/ncu_summary.py report.ncu-rep [source-note]"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_us",
    "dram__bytes_read.sum": "dram_read_MB",
    "dram__bytes_write.sum": "dram_write_MB",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_theoretical",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_active_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_rate_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
}
rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h, units = rows[0], rows[1]
out = []
for r in rows[2:]:
    d = {"kernel": r[h.index("Kernel Name")][:80]}
    for k, name in KEYS.items():
        if k in h:
            i = h.index(k)
            v = float(r[i].replace(",", ""))
            u = units[i]
            if name.endswith("_MB"):
                v = v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
            if name == "duration_us":
                v = v * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3,
                         "msecond": 1e3}.get(u, 1.0)
            d[name] = round(v, 4)
    if "dram_read_MB" in d and "duration_us" in d:
        d["dram_TBps"] = round((d["dram_read_MB"] + d["dram_write_MB"]) / d["duration_us"], 4)
    out.append(d)
print(json.dumps({"source": sys.argv[2] if len(sys.argv) > 2 else rep, "launches": out}, indent=1))
