"""Aggregate an ncu '--page source --print-source cuda,sass --csv' dump per CUDA source
line: executed instructions and stall samples.  Usage: ncu_line_summary.py file.csv [N]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
inst = collections.Counter()
stall = collections.Counter()
text = {}
cur_file = ""
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    try:
        ln = r[0]
        key = (cur_file, int(ln)) if ln else None
    except ValueError:
        continue
    if key is None:
        continue
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ii = hdr.index("Instructions Executed")
    try:
        s = float(r[si] or 0)
        n = float(r[ii] or 0)
    except ValueError:
        continue
    inst[key] += n
    stall[key] += s
    text[key] = r[1]
ti = sum(inst.values()) or 1
ts = sum(stall.values()) or 1
print(f"instructions {ti:.3e}  stall samples {ts:.0f}")
for key, n in inst.most_common(top):
    print(f"{n / ti * 100:6.2f}% inst {stall[key] / ts * 100:6.2f}% stall  {key[0]}:{key[1]}  {text[key].strip()[:80]}")
