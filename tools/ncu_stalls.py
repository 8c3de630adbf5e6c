"""Aggregate an `ncu --page source --csv` export by opcode: executed count,
stall samples by reason, and the instructions with the most samples.

usage: ncu -i rep.ncu-rep --page source --csv > src.csv; python tools/ncu_stalls.py src.csv
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hi]
ix = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows[hi + 1:]:  # the first kernel of the export
    if r and r[0] == "Kernel Name":
        break
    if len(r) == len(hdr) and r[0].startswith("0x"):
        data.append(r)
keys = ("stall_wait", "stall_long_sb", "stall_math", "stall_short_sb", "stall_selected",
        "stall_not_selected", "stall_branch_resolving", "stall_barrier")
tot = sum(int(r[ix["# Samples"]]) for r in data)
print("total samples", tot)
agg = defaultdict(lambda: defaultdict(int))
for r in data:
    src = r[ix["Source"]].split()
    op = (src[1] if src[0].startswith("@") else src[0]).split(".")[0]
    for k in ("# Samples",) + keys:
        agg[op][k] += int(r[ix[k]])
    agg[op]["n"] += int(r[ix["Instructions Executed"]])
print("%-8s %10s %8s " % ("op", "executed", "samples") + " ".join("%8s" % k[6:14] for k in keys))
for op, a in sorted(agg.items(), key=lambda x: -x[1]["# Samples"])[:16]:
    print("%-8s %10d %8d " % (op, a["n"], a["# Samples"]) + " ".join("%8d" % a[k] for k in keys))
print()
for r in sorted(data, key=lambda r: -int(r[ix["# Samples"]]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print("%6s  %-64s " % (r[ix["# Samples"]], " ".join(r[ix["Source"]].split())[:64]) +
          " ".join("%s=%s" % (k[6:], r[ix[k]]) for k in keys if int(r[ix[k]]) > 0))
