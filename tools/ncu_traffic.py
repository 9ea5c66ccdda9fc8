"""Summarise an ncu --set full report (read here, no GPU) into
profiles/ncu_traffic.json: per kernel name, DRAM bytes per launch, duration,
DRAM throughput %.

    python tools/ncu_traffic.py gpurun_out/prof_mv.ncu-rep U32k
"""
import csv
import io
import json
import os
import subprocess
import sys

rep, tag = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
want = ["Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active"]
idx = {w: hdr.index(w) for w in want if w in hdr}
units = rows[1]
res = {}
for r in rows[2:]:
    name = r[idx["Kernel Name"]].split("(")[0].split("::")[-1]
    def val(k):
        v = r[idx[k]].replace(",", "")
        u = units[idx[k]]
        x = float(v)
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                 "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}.get(u, 1)
        return x * scale
    ent = res.setdefault(name, [])
    ent.append({"dram_bytes": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
                "duration_s": val("gpu__time_duration.sum"),
                "dram_pct": val("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                "regs": val("launch__registers_per_thread")})
summary = {k: {"traffic_bytes_per_launch": sum(e["dram_bytes"] for e in v) / len(v),
               "duration_ms": 1e3 * sum(e["duration_s"] for e in v) / len(v),
               "dram_pct_of_peak": sum(e["dram_pct"] for e in v) / len(v), "launches": len(v),
               "registers": v[0]["regs"]} for k, v in res.items()}
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
data = json.load(open(path)) if os.path.exists(path) else {}
data[tag] = {k: v["traffic_bytes_per_launch"] for k, v in summary.items()}
data.setdefault("_detail", {})[tag] = summary
json.dump(data, open(path, "w"), indent=1)
print(json.dumps(summary, indent=1))
