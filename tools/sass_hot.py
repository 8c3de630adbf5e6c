"""Per-opcode instruction / stall-sample shares and the hottest SASS lines of
the first kernel in an ncu report (source page).

usage: python tools/sass_hot.py report.ncu-rep [kernel-regex] [top]
"""
import csv
import io
import subprocess
import sys
from collections import Counter, defaultdict

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else None
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if kre:
    cmd += ["-k", "regex:" + kre]
rows = list(csv.reader(io.StringIO(subprocess.run(cmd, capture_output=True, text=True).stdout)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = []
        blocks.append(cur)
        continue
    if cur is not None:
        cur.append(r)
b = blocks[0]
h = b[0]
data = [r for r in b[1:] if len(r) == len(h)]
ix = {k: i for i, k in enumerate(h)}


def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


S = "Warp Stall Sampling (All Samples)"
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot_s = sum(num(r[ix[S]]) for r in data)
tot_i = sum(num(r[ix["Instructions Executed"]]) for r in data)
c, cs = Counter(), Counter()
why = defaultdict(Counter)
for r in data:
    t = r[ix["Source"]].split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") else t[0]
    op = op if op.startswith(("LD", "ST")) else op.split(".")[0]
    c[op] += num(r[ix["Instructions Executed"]])
    cs[op] += num(r[ix[S]])
    for s in stalls:
        why[op][s] += num(r[ix[s]])
print(f"instructions {tot_i:.4g}, samples {tot_s:.4g}")
for op, v in c.most_common(top):
    w = ", ".join(f"{s[6:]} {x / max(tot_s, 1) * 100:.1f}" for s, x in why[op].most_common(3))
    print(f"{op:26s} {v / tot_i * 100:5.1f}% inst {cs[op] / tot_s * 100:5.1f}% samples  ({w})")
print("-- hottest lines by samples")
for r in sorted(data, key=lambda r: -num(r[ix[S]]))[:top]:
    print(f"{r[ix['Address']]:>8s} {num(r[ix[S]]) / tot_s * 100:5.2f}%  {r[ix['Source']][:90]}")
