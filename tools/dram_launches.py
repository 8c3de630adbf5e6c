"""profiles/ncu_summary.json from an ncu launch list with DRAM bytes
(`ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
--csv --log-file X.csv`): per launch the kernel, DRAM read / write bytes and
duration.  bench.py reads it for roofline.traffic.

usage: python tools/dram_launches.py profiles/rNN/dram_c2_all_launches.csv "<source note>"
"""
import csv
import json
import os
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hi]
ix = {k: i for i, k in enumerate(h)}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3,
         "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
KEY = {"dram__bytes_read.sum": "dram_read_bytes", "dram__bytes_write.sum": "dram_write_bytes",
       "gpu__time_duration.sum": "duration_us"}
launches = {}
for r in rows[hi + 1:]:
    if len(r) != len(h) or r[ix["Metric Name"]] not in KEY:
        continue
    name = re.sub(r"\(.*", "", r[ix["Kernel Name"]])
    m = re.search(r"(k_\w+.*)$", name)  # drop "void ifgf_b200::<unnamed>::"
    name = m.group(1) if m else name
    rec = launches.setdefault(r[ix["ID"]], {"id": r[ix["ID"]], "kernel": name})
    v = float(r[ix["Metric Value"]].replace(",", "")) * SCALE.get(r[ix["Metric Unit"]], 1.0)
    rec[KEY[r[ix["Metric Name"]]]] = v
out = {"source": sys.argv[2] if len(sys.argv) > 2 else sys.argv[1],
       "launches": list(launches.values())}
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
json.dump(out, open(os.path.join(root, "profiles", "ncu_summary.json"), "w"), indent=0)
for rec in out["launches"]:
    print(f"{rec['kernel'][:44]:44s} {rec.get('duration_us', 0) / 1e3:8.3f} ms  "
          f"read {rec.get('dram_read_bytes', 0) / 1e9:7.3f} GB  write {rec.get('dram_write_bytes', 0) / 1e9:6.3f} GB")
