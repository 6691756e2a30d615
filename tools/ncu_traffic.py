"""DRAM traffic of the bin-rasterizer kernels of one frame from an ncu capture.

usage: python tools/ncu_traffic.py report.ncu-rep workload [profiles/traffic.json]

The capture must hold exactly one frame's k_extract / k_shade / k_finalize
launches (tools/profile_frame.py + ncu -k regex + --launch-skip/-count).
Writes {workload: {"raster_dram_bytes": R+W summed, "kernels": [...]}} into
the JSON file that bench.py reads for roofline.traffic.
"""
import csv
import io
import json
import subprocess
import sys

rep, workload = sys.argv[1], sys.argv[2]
out_path = sys.argv[3] if len(sys.argv) > 3 else "profiles/traffic.json"
metrics = ("dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
           "smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum")
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", metrics],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, units, data = rows[0], rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}


def val(r, name):
    v = float(r[ix[name]].replace(",", "") or 0)
    u = units[ix[name]]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
             "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}
    return v * scale.get(u, 1)


kernels = []
for r in data:
    name = r[ix["Kernel Name"]]
    kernels.append({"kernel": name.split("(")[0],
                    "dram_read_bytes": val(r, "dram__bytes_read.sum"),
                    "dram_write_bytes": val(r, "dram__bytes_write.sum"),
                    "ncu_ms": val(r, "gpu__time_duration.sum"),
                    "issue_active_pct": val(r, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                    "warp_instructions": val(r, "smsp__inst_executed.sum")})
total = sum(k["dram_read_bytes"] + k["dram_write_bytes"] for k in kernels)
try:
    with open(out_path) as f:
        doc = json.load(f)
except (OSError, ValueError):
    doc = {}
top = max(kernels, key=lambda k: k["ncu_ms"])
doc[workload] = {"raster_dram_bytes": total, "kernels": kernels, "source": rep.split("/")[-1],
                 "top_kernel": top["kernel"], "top_issue_active_pct": top["issue_active_pct"]}
with open(out_path, "w") as f:
    json.dump(doc, f, indent=1)
print(json.dumps(doc[workload], indent=1))
