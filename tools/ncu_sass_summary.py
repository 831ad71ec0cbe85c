"""Summarise an ncu --page source --csv (SASS) dump: top instructions by stall
samples and executed-instruction mix by opcode.  Usage: ncu_sass_summary.py file.csv [N]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
h = next(i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r)
hdr = rows[h]
si = hdr.index("Warp Stall Sampling (All Samples)")
ii = hdr.index("Instructions Executed")
src = hdr.index("Source")
data = []
for r in rows[h + 1:]:
    try:
        data.append((float(r[si] or 0), float(r[ii] or 0), r[0], r[src]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
toti = sum(d[1] for d in data) or 1
print(f"total stall samples {tot:.0f}, instructions {toti:.3e}")
ops = collections.Counter()
opstall = collections.Counter()
for s, n, a, t in data:
    op = t.split()[0] if t.split() else "?"
    if op.startswith("@"):
        op = t.split()[1]
    op = op.split(".")[0]
    ops[op] += n
    opstall[op] += s
print("opcode mix (inst %, stall %):")
for op, n in ops.most_common(25):
    print(f"  {op:10s} {n / toti * 100:6.2f}%  {opstall[op] / tot * 100:6.2f}%")
print("top instructions by stall samples:")
for s, n, a, t in sorted(data, reverse=True)[:top]:
    print(f"  {s / tot * 100:5.2f}% {n / toti * 100:5.2f}%  {a}: {t[:90]}")
