#!/usr/bin/env python
"""profiles/traffic.json <- dram__bytes_read.sum + dram__bytes_write.sum of the first kernel in
an `ncu --set full` report (bench.py reads it for roofline.traffic).
usage: python tools/update_traffic.py REPORT.ncu-rep CONFIG KEY [NOTE]"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, cfg, key = sys.argv[1], sys.argv[2], sys.argv[3]
note = sys.argv[4] if len(sys.argv) > 4 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units, v = rows[0], rows[1], rows[2]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
tot = 0.0
for name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
    i = h.index(name)
    tot += float(v[i].replace(",", "")) * scale[units[i]]
path = os.path.join(ROOT, "profiles", "traffic.json")
t = json.load(open(path))
t.setdefault(f"config{cfg}", {})[key] = int(tot)
t["_about"] = (t.get("_about", "") + f" | config{cfg} {key}: {tot / 1e9:.3f} GB from {os.path.basename(rep)} "
               f"{v[h.index('Kernel Name')][:60]} {note}").strip(" |")
json.dump(t, open(path, "w"), indent=1)
print(f"config{cfg} {key} = {tot / 1e9:.3f} GB")
