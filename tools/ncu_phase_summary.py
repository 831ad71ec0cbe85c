"""Stall samples and executed instructions of one kernel grouped by source-line
ranges (phases).  Usage: ncu_phase_summary.py source.csv file.cu 'name:start_marker' ...
(each phase runs from its marker line to the line before the next marker)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
fname = sys.argv[2].split("/")[-1]
src = open(sys.argv[2]).read().split("\n")
marks = []
for spec in sys.argv[3:]:
    name, m = spec.split(":", 1)
    ln = next(i + 1 for i, l in enumerate(src) if m in l)
    marks.append((ln, name))
marks.sort()
hdr, cur = None, ""
inst, st = collections.Counter(), collections.Counter()
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    try:
        ln = int(r[0])
        s = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        n = float(r[hdr.index("Instructions Executed")] or 0)
    except ValueError:
        continue
    inst[(cur, ln)] += n
    st[(cur, ln)] += s
ts, ti = sum(st.values()) or 1, sum(inst.values()) or 1
bounds = marks + [(10 ** 9, None)]
for (a, name), (b, _) in zip(bounds[:-1], bounds[1:]):
    s = sum(v for (f, l), v in st.items() if f == fname and a <= l < b)
    i = sum(v for (f, l), v in inst.items() if f == fname and a <= l < b)
    print(f"{name:24s} lines {a:4d}-{b - 1 if b < 10 ** 9 else 'end'}: stall {100 * s / ts:5.1f}%  inst {100 * i / ti:5.1f}%")
for f in sorted({f for (f, _) in st} - {fname}):
    print(f"{f:24s} stall {100 * sum(v for (g, _), v in st.items() if g == f) / ts:5.1f}%")
