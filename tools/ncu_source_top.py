"""Summarise an ncu `--page source --csv --print-source sass` export: the
instructions with the most warp-stall samples and the executed-instruction
histogram by opcode (which SASS the kernel spends its issue slots on).

    python tools/ncu_source_top.py gpurun_out/<name>_source.csv [N]
"""
import collections
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
hdr = rows[1]
ix = {k: i for i, k in enumerate(hdr)}
recs = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    recs.append(r)
samples = lambda r: int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
execd = lambda r: int(r[ix["Instructions Executed"]] or 0)
tot_s = sum(samples(r) for r in recs)
tot_e = sum(execd(r) for r in recs)
print(f"total samples {tot_s}, warp instructions executed {tot_e}")
ops = collections.Counter()
for r in recs:
    src = r[ix["Source"]].strip()
    tok = src.split()
    op = tok[0] if tok else "?"
    if op.startswith("@"):
        op = tok[1] if len(tok) > 1 else op
    ops[op.split(".")[0]] += execd(r)
print("executed by opcode:")
for op, n in ops.most_common(25):
    print(f"  {op:12s} {n:14d} {100.0 * n / max(tot_e, 1):5.1f}%")
stall_cols = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
print(f"top {top} instructions by stall samples:")
for r in sorted(recs, key=samples, reverse=True)[:top]:
    st = sorted(((int(r[ix[c]] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
    print(f"  {r[ix['Address']][-5:]} {samples(r):6d} {execd(r):11d}  {r[ix['Source']].strip()[:60]:60s} {st}")
