"""One-screen summary of an ncu --set full report (raw page CSV) per kernel launch:
duration, DRAM bytes, FP64/DMMA pipe, L1 wavefronts, occupancy, issue and stall ratios.
Usage: ncu -i rep.ncu-rep --page raw --csv > raw.csv; ncu_kernel_summary.py raw.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, units = rows[0], rows[1]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "smsp__issue_active.avg.pct_of_peak_sustained_active"]
STALL = "smsp__average_warps_issue_stalled_"
for r in rows[2:]:
    print("==", r[hdr.index("Kernel Name")][:110])
    for k in KEYS:
        if k in hdr:
            print(f"   {k:78s} {r[hdr.index(k)]:>14s} {units[hdr.index(k)]}")
    st = [(h[len(STALL):].replace("_per_issue_active.ratio", ""), float(r[i] or 0))
          for i, h in enumerate(hdr) if h.startswith(STALL) and h.endswith("per_issue_active.ratio")]
    st = [x for x in sorted(st, key=lambda x: -x[1]) if x[1] >= 0.1]
    print("   stalls/issue: " + ", ".join(f"{a} {b:.2f}" for a, b in st))
