"""Aggregate an ncu source page (SASS rows) by stall reason and by code
region: python scripts/ncu_stalls.py report.ncu-rep"""
import collections
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]
data = [r for r in rows[hi + 1:] if r and r[0].startswith("0x")]
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = collections.Counter()
for r in data:
    for c in reasons:
        v = r[h.index(c)]
        tot[c] += int(v) if v else 0
s = sum(tot.values())
print("stall samples by reason:")
for c, v in tot.most_common():
    if v:
        print(f"  {c:24s} {v:7d} {100*v/s:5.1f}%")
ie = h.index("Instructions Executed")
ops = collections.Counter()
for r in data:
    src = r[h.index("Source")].split()
    if not src:
        continue
    op = src[1] if src[0].startswith("@") else src[0]
    ops[op.split(".")[0]] += int(r[ie] or 0)
n = sum(ops.values())
print(f"warp instructions executed: {n}")
for op, v in ops.most_common(15):
    print(f"  {op:10s} {v:10d} {100*v/n:5.1f}%")
