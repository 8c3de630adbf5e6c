"""Attribute executed SASS instructions (from an ncu source-page CSV) to CUDA
source lines / inlined functions using nvdisasm line info of the same cubin.

usage: python tools/sass_lines.py <obj.o> <kernel-substring> <ncu_sass.csv>
(ncu_sass.csv: `ncu -i rep --page source --csv --print-source sass -k ...`)
"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile


def sass_with_lines(obj, kname):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, check=True,
                   capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True,
                         text=True).stdout
    out, inside, line, fn = [], False, None, None
    for l in txt.splitlines():
        if l.strip().startswith(".section") and ".text." in l:
            inside = kname in l
            continue
        if not inside:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)(.*inlined at "([^"]+)", line (\d+))?', l)
        if m:
            line = (os.path.basename(m.group(1)), int(m.group(2)))
            fn = (os.path.basename(m.group(4)), int(m.group(5))) if m.group(4) else None
            continue
        m = re.match(r"\s*/\*([0-9a-f]+)\*/\s+(.*?);", l)
        if m:
            out.append((int(m.group(1), 16), m.group(2).strip(), line, fn))
    return out


def main(obj, kname, csvp):
    sass = sass_with_lines(obj, kname)
    rows = list(csv.reader(open(csvp)))
    hdr = rows[1]
    iex = hdr.index("Instructions Executed")
    ist = hdr.index("Warp Stall Sampling (All Samples)")
    ex = []
    for r in rows[2:]:
        try:
            ex.append((int(r[iex]), int(r[ist]), r[1].strip()))
        except Exception:
            pass
    # ncu lists each instruction once per address; align by order
    n = min(len(ex), len(sass))
    by_line = collections.Counter()
    st_line = collections.Counter()
    fp64 = collections.Counter()
    for (e, s, src), (addr, ins, line, fn) in zip(ex[:n], sass[:n]):
        key = f"{line[0]}:{line[1]}" if line else "?"
        by_line[key] += e
        st_line[key] += s
        if re.match(r"(@\S+\s+)?D(FMA|ADD|MUL|SETP|MNMX)", ins):
            fp64[key] += e
    tot = sum(by_line.values())
    print(f"aligned {n} of ncu {len(ex)} / sass {len(sass)}; executed warp-instrs {tot}")
    for k, v in by_line.most_common(45):
        print(f"{v:>12d} {100 * v / tot:5.1f}%  fp64 {fp64[k]:>11d}  stalls {st_line[k]:>7d}  {k}")


if __name__ == "__main__":
    main(*sys.argv[1:4])
