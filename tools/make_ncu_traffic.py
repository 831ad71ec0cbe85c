"""Build profiles/ncu_traffic.json (read by bench.py for roofline.traffic and the executed
FP64 fractions) from ncu captures: per workload and kernel, the mean per launch of
dram__bytes_read.sum + dram__bytes_write.sum, the DMMA pipe and FP64 pipe activity.
Usage: make_ncu_traffic.py out.json workload1=capture1.csv [workload2=raw2.csv ...]
(capture = `--metrics ... --csv` launch list or `--page raw --csv` export)."""
import collections
import csv
import json
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "%": 1, "ns": 1, "nsecond": 1,
        "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}


def load(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    rows = list(csv.reader(lines))
    acc = collections.defaultdict(lambda: collections.defaultdict(list))
    if rows and "Metric Name" in rows[0]:  # launch-list format: one row per metric
        h = rows[0]
        for r in rows[1:]:
            d = dict(zip(h, r))
            k = d["Kernel Name"].split("(")[0].replace("void ", "").replace("rbf::", "")
            acc[k][d["Metric Name"]].append(float(d["Metric Value"].replace(",", "")) *
                                             UNIT.get(d["Metric Unit"], 1))
    else:  # raw page: header row, unit row, one row per launch
        h, u = rows[0], rows[1]
        for r in rows[2:]:
            k = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("rbf::", "")
            for name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                         "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
                         "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"):
                if name in h and r[h.index(name)]:
                    acc[k][name].append(float(r[h.index(name)].replace(",", "")) * UNIT.get(u[h.index(name)], 1))
    out = {}
    for k, m in acc.items():
        mean = {n: sum(v) / len(v) for n, v in m.items()}
        e = {"launches_captured": max(len(v) for v in m.values())}
        if "dram__bytes_read.sum" in mean:
            e["dram_bytes_per_launch"] = mean["dram__bytes_read.sum"] + mean.get("dram__bytes_write.sum", 0.0)
        if "gpu__time_duration.sum" in mean:
            e["ms_per_launch_ncu"] = mean["gpu__time_duration.sum"] / 1e6
        t = mean.get("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active")
        if t is not None:
            e["fp64_tensor_pct_of_peak"] = t
        f = mean.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")
        if f is not None:
            e["fp64_pipe_pct_of_peak"] = f
        out[k] = e
    return out


res = {}
for arg in sys.argv[2:]:
    wl, path = arg.split("=", 1)
    res[wl] = load(path)
    res[wl]["_source"] = path
json.dump(res, open(sys.argv[1], "w"), indent=1)
print(json.dumps(res, indent=1)[:3000])
