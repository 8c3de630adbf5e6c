"""Per-kernel share of an ncu launch list (`--metrics gpu__time_duration.sum
--csv --log-file ...`): launches, summed duration and share, one line per
kernel.  Per-launch ncu times are serialised and cold-cache, so compare
shares, not absolute times.

usage: python tools/launch_share.py launches.csv [out.txt]
"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hi]
ix = {k: i for i, k in enumerate(h)}
tot, cnt = collections.Counter(), collections.Counter()
for r in rows[hi + 1:]:
    if len(r) != len(h) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = r[ix["Kernel Name"]].replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    name = re.sub(r"\(.*", "", name).replace("void ", "")
    name = re.sub(r"^.*::", "", re.sub(r"<.*", "", name)) + (
        re.search(r"<.*>", name).group(0) if "<" in name else "")
    v = float(r[ix["Metric Value"]].replace(",", ""))
    v *= {"ns": 1e-3, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(r[ix["Metric Unit"]], 1.0)
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
lines = [f"{'kernel':56s} {'launches':>8s} {'ms':>10s} {'share':>7s}"]
for k, v in tot.most_common():
    lines.append(f"{k[:56]:56s} {cnt[k]:8d} {v / 1e3:10.3f} {v / T * 100:6.2f}%")
lines.append(f"{'total':56s} {sum(cnt.values()):8d} {T / 1e3:10.3f}")
out = "\n".join(lines)
print(out)
if len(sys.argv) > 2:
    open(sys.argv[2], "w").write(out + "\n")
