"""Attribute an ncu SASS source-page CSV to CUDA source lines.

usage: sass_lines.py <ncu-sass.csv> <nvdisasm -g -c output> <function symbol> [top]
The ncu CSV comes from `ncu -i rep --page source --csv --print-source sass`, the
disassembly from `nvdisasm -g -c <cubin>` of the same build (-lineinfo)."""
import collections
import csv
import re
import sys

csv_path, sass_path, fun = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
# offset -> line from the disassembly
off2line = {}
cur = None
infun = False
for ln in open(sass_path):
    if ln.startswith("//---------------------"):
        infun = fun in ln
        continue
    if not infun:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        off2line[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(csv_path)))
h = rows[1]
ci, cw, cs = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
data = []
for r in rows[2:]:
    if len(r) <= ci:
        continue
    try:
        data.append((int(r[0], 16), int(float(r[ci] or 0)), int(float(r[cw] or 0)), r[cs]))
    except ValueError:
        pass
base = min(d[0] for d in data)
inst = collections.Counter()
stall = collections.Counter()
for a, n, w, s in data:
    key = off2line.get(a - base, ("?", 0))
    inst[key] += n
    stall[key] += w
ti, tw = sum(inst.values()), sum(stall.values())
print(f"total inst {ti:.3e} samples {tw}")
for key, n in sorted(inst.items(), key=lambda kv: -stall[kv[0]])[:top]:
    print(f"{key[0]}:{key[1]:<5d} inst {n / ti * 100:5.1f}%  stall {stall[key] / tw * 100:5.1f}%")

# stall reasons per top line
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
ri = [h.index(c) for c in reasons]
per = collections.defaultdict(collections.Counter)
tot_r = collections.Counter()
for r in rows[2:]:
    if len(r) <= max(ri):
        continue
    try:
        a = int(r[0], 16)
    except ValueError:
        continue
    key = off2line.get(a - base, ("?", 0))
    for c, i in zip(reasons, ri):
        v = int(float(r[i] or 0))
        per[key][c] += v
        tot_r[c] += v
print("stall reasons (all):", ", ".join(f"{c[6:]} {v / tw * 100:.1f}%" for c, v in tot_r.most_common(8)))
for key, n in sorted(inst.items(), key=lambda kv: -stall[kv[0]])[:12]:
    print(f"{key[0]}:{key[1]:<5d}", ", ".join(f"{c[6:]} {v / tw * 100:.1f}" for c, v in per[key].most_common(4)))
