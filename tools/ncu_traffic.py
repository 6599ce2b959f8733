"""Write the per-layer DRAM traffic of the grouped FFN launches of an ncu --set full
capture (tools/ffn_probe.py at a bench shape) into profiles/<round>/ffn_traffic.json,
the file bench.py stamps into roofline.traffic.

    python tools/ncu_traffic.py rep.ncu-rep key out.json "<how the capture was taken>"
"""
import csv
import io
import json
import os
import subprocess
import sys

rep, key, out, how = sys.argv[1:5]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]


def val(r, name):
    i = hdr.index(name)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "nsecond": 1e-3,
             "msecond": 1e3}.get(units[i], 1)
    return float(r[i].replace(",", "")) * scale


kern = {}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
    kern.setdefault(name, {"dram_read_bytes": val(r, "dram__bytes_read.sum"),
                           "dram_write_bytes": val(r, "dram__bytes_write.sum"),
                           "gpu_time_us": val(r, "gpu__time_duration.sum")})
tot = sum(k["dram_read_bytes"] + k["dram_write_bytes"] for k in kern.values())
data = json.load(open(out)) if os.path.exists(out) else {}
data[key] = {"source": how, "kernels": kern, "dram_bytes_per_layer": tot}
json.dump(data, open(out, "w"), indent=1)
print(json.dumps(data[key], indent=1))
