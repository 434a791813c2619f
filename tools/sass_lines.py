"""Attribute ncu SASS-level warp-stall samples to CUDA source lines.
usage: sass_lines.py <ncu source-page csv (SASS)> <nvdisasm -g -c output> [kernel mangled name]"""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
h = rows[hi]
si = h.index("Warp Stall Sampling (All Samples)")
samples = []
for r in rows[hi + 1:]:
    try:
        samples.append((int(r[0], 16), int(r[si])))
    except Exception:
        pass
base = samples[0][0]
# nvdisasm -g: lines "//## File ..., line N" precede instructions "/*0a30*/"
fn = sys.argv[3] if len(sys.argv) > 3 else None
cur = None
infn = fn is None
line_of = {}
for ln in open(sys.argv[2]):
    if fn and ".text." in ln and ln.strip().startswith(".section"):
        infn = fn in ln
    m = re.search(r'//## File ".*?([^/"]+)", line (\d+)', ln)
    if m:
        cur = f"{m.group(1)}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and infn:
        line_of[int(m.group(1), 16)] = cur
agg = defaultdict(int)
for a, n in samples:
    agg[line_of.get(a - base, "?")] += n
tot = sum(agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:int(sys.argv[4]) if len(sys.argv) > 4 else 40]:
    print(f"{100.0 * v / tot:5.1f}%  {k}")
