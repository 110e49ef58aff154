"""Summarise an ncu launch list (gpu__time_duration per launch) and a --set full
report into markdown for profiles/.  Usage:
  python tools/ncu_summary.py launches.csv [report.ncu-rep] > profiles/rNN_....md"""
import collections
import csv
import io
import subprocess
import sys

UNITS = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        tot[name] += float(r[vi].replace(",", "")) * UNITS.get(r[ui], 1.0)
        cnt[name] += 1
    T = sum(tot.values())
    print(f"### Launch list ({sum(cnt.values())} launches, {T:.3f} ms serialized, cold-cache)\n")
    print("| kernel | launches | ms total | share |\n|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"| `{k}` | {cnt[k]} | {v:.3f} | {100 * v / T:.1f}% |")
    print()


METRICS = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "DRAM read"),
           ("dram__bytes_write.sum", "DRAM write"), ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
           ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
           ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
           ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
           ("launch__registers_per_thread", "regs"), ("launch__occupancy_limit_registers", "occ limit regs")]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    idx = [(hdr.index(m), lab) for m, lab in METRICS if m in hdr]
    ki = hdr.index("Kernel Name")
    print("### ncu --set full (per launch)\n")
    print("| kernel | " + " | ".join(f"{lab} [{units[i]}]" for i, lab in idx) + " |")
    print("|---|" + "---|" * len(idx))
    for r in rows[2:]:
        print(f"| `{r[ki][:60]}` | " + " | ".join(r[i] for i, _ in idx) + " |")
    print()


if __name__ == "__main__":
    launches(sys.argv[1])
    if len(sys.argv) > 2:
        full(sys.argv[2])
