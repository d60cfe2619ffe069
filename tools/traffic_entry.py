"""Adds one kernel's per-launch DRAM bytes and warp instructions per extension, read from an
`ncu --set full` report (here, no GPU), to profiles/traffic.json -- what bench.py reports as the
roofline's `traffic` and its issue-slot view.

usage: python tools/traffic_entry.py <rep> <key> <extensions of the launch> <source .md> [launch index]"""
import csv
import io
import json
import os
import subprocess
import sys

rep, key, ext, src = sys.argv[1], sys.argv[2], float(sys.argv[3]), sys.argv[4]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
vals = rows[2 + (int(sys.argv[5]) if len(sys.argv) > 5 else 0)]  # the profiled launch
d = dict(zip(hdr, vals))
u = dict(zip(hdr, units))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rd = float(d["dram__bytes_read.sum"].replace(",", "")) * scale.get(u["dram__bytes_read.sum"], 1)
wr = float(d["dram__bytes_write.sum"].replace(",", "")) * scale.get(u["dram__bytes_write.sum"], 1)
inst = float(d["smsp__inst_executed.sum"].replace(",", ""))
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
try:
    with open(path) as f:
        t = json.load(f)
except Exception:
    t = {}
t[key] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr, "warp_inst_per_launch": inst,
          "extensions_per_launch": ext, "warp_inst_per_ext": inst / ext if ext else None, "source": src,
          "kernel": d.get("Kernel Name", "")[:120]}
with open(path, "w") as f:
    json.dump(t, f, indent=1)
print(key, t[key])
