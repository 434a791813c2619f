"""Per-source-line warp-stall samples by reason from an ncu source page (SASS, csv) and the
nvdisasm -g -c listing of the same cubin.
usage: stall_lines.py <csv> <nvdisasm listing> <kernel substring> [top] [reason]"""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
h = rows[hi]
reasons = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
idx = {x: h.index(x) for x in reasons}
fn = sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
sel = sys.argv[5] if len(sys.argv) > 5 else None
data = []
for r in rows[hi + 1:]:
    try:
        data.append((int(r[0], 16), {k: int(r[i]) for k, i in idx.items()}))
    except Exception:
        pass
base = data[0][0]
cur, infn, line_of = None, False, {}
for ln in open(sys.argv[2]):
    if ".text." in ln and ln.strip().startswith(".section"):
        infn = fn in ln
    m = re.search(r'//## File ".*?([^/"]+)", line (\d+)', ln)
    if m:
        cur = f"{m.group(1)}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and infn:
        line_of[int(m.group(1), 16)] = cur
agg = defaultdict(lambda: defaultdict(int))
tot = defaultdict(int)
for a, d in data:
    ln = line_of.get(a - base, "?")
    for k, v in d.items():
        agg[ln][k] += v
        tot[k] += v
T = sum(tot.values())
print("reasons:", " ".join(f"{k[6:]}={100.0 * v / T:.1f}%" for k, v in sorted(tot.items(), key=lambda kv: -kv[1]) if v))
key = (lambda kv: -kv[1][sel]) if sel else (lambda kv: -sum(kv[1].values()))
for ln, d in sorted(agg.items(), key=key)[:top]:
    s = sum(d.values())
    parts = " ".join(f"{k[6:]}={v}" for k, v in sorted(d.items(), key=lambda kv: -kv[1])[:4] if v)
    print(f"{100.0 * s / T:5.1f}%  {ln:28s} {parts}")
