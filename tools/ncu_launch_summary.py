"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel:
launches, total and mean device time, share.  Usage: ncu_launch_summary.py launches.csv"""
import collections
import csv
import sys

lines = [l for l in open(sys.argv[1]) if not l.startswith("==")]
d = collections.defaultdict(lambda: [0, 0.0])
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    k = r["Kernel Name"].split("(")[0].replace("void ", "")
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(r["Metric Unit"], 1e-6)
    d[k][0] += 1
    d[k][1] += float(r["Metric Value"].replace(",", "")) * scale
tot = sum(v[1] for v in d.values())
print(f"{'kernel':64s} {'launches':>8s} {'total ms':>10s} {'mean us':>9s} {'share':>6s}")
for k, v in sorted(d.items(), key=lambda x: -x[1][1]):
    print(f"{k[:64]:64s} {v[0]:8d} {v[1]:10.3f} {1e3 * v[1] / v[0]:9.1f} {100 * v[1] / tot:5.1f}%")
print(f"{'TOTAL':64s} {sum(v[0] for v in d.values()):8d} {tot:10.3f}")
