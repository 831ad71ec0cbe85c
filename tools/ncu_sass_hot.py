"""Hottest SASS instructions of an ncu '--page source --print-source cuda,sass --csv' dump
with their source line and main stall reasons.  Usage: ncu_sass_hot.py file.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None
cur = None
out = []
tot = 0
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if len(r) > 3 and r[0] and r[0].isdigit():
        cur = int(r[0])
        continue
    if len(r) > 7 and r[2].startswith("0x"):
        s = int(r[4] or 0)
        tot += s
        st = {hdr[k][6:]: int(r[k] or 0) for k in range(len(hdr)) if hdr[k].startswith("stall_") and "Not Issued" not in hdr[k]}
        out.append((s, r[2][-5:], cur, r[3].strip()[:60], st))
out.sort(key=lambda x: -x[0])
print(f"stall samples {tot}")
for s, a, line, ins, st in out[:top]:
    main = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{100 * s / tot:5.1f}% {a} L{line} {ins:60s} " + " ".join(f"{k}:{v}" for k, v in main if v))
