"""Key metrics from `ncu --page raw --csv` exports: python tools/ncu_csv_summary.py a.csv [b.csv ...]"""
import csv
import sys

KEYS = ["Kernel Name", "gpu__time_duration.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "dram__bytes_read.sum", "dram__bytes_write.sum"]
for path in sys.argv[1:]:
    r = list(csv.reader(open(path)))
    hdr = r[0]
    print("==", path)
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            print("  " + k[:70].ljust(70), [x[i][:50] for x in r[2:]])
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
            v = [x[i] for x in r[2:]]
            if max(float(a or 0) for a in v) > 0.1:
                print("  stall " + h[34:-23].ljust(64), v)
