"""Aggregate ncu warp-stall samples and executed instructions by CUDA source
line: `ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > f.csv`
then `python tools/ncu_lines.py f.csv [top]`."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
agg = collections.defaultdict(lambda: [0.0, 0.0])
fname, cur, tot = None, None, 0.0
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] == "Line No":
        continue
    try:
        s, ie = float(r[4] or 0), float(r[7] or 0)
    except ValueError:
        continue
    if r[0]:
        cur = (fname, r[0], r[1].strip()[:90])
    agg[cur][0] += s
    agg[cur][1] += ie
    tot += s
print("total samples", tot)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{int(v[0]):7d} {100 * v[0] / tot:5.1f}%  {k[0]}:{k[1]:>4}  {int(v[1]):>11}  {k[2]}")
