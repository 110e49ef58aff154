"""Summarise an ncu launch list (gpu__time_duration per launch) and --set full
reports into markdown for profiles/, and (--traffic out.json) the per-launch
DRAM traffic of the captured kernels that bench.py reports.  Usage:
  python tools/ncu_summary.py launches.csv [report.ncu-rep ...] [--traffic profiles/rNN_ncu_traffic_c2.json]"""
import collections
import csv
import io
import json
import re
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
        name = r[ki].split("(")[0].replace("void ", "").replace("igb::dev::", "")
        tot[name] += float(r[vi].replace(",", "")) * UNITS.get(r[ui], 1.0)
        cnt[name] += 1
    T = sum(tot.values())
    print(f"### Launch list ({sum(cnt.values())} launches, {T:.3f} ms serialized, cold-cache)\n")
    print("| kernel | launches | ms total | us / launch | share |\n|---|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"| `{k}` | {cnt[k]} | {v:.3f} | {1e3 * v / cnt[k]:.1f} | {100 * v / T:.1f}% |")
    print()


METRICS = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "DRAM read"),
           ("dram__bytes_write.sum", "DRAM write"), ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
           ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
           ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
           ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
           ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
           ("launch__registers_per_thread", "regs"), ("launch__occupancy_limit_registers", "occ limit regs")]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def short(name):
    name = name.replace("igb::dev::", "").replace("void ", "")
    return re.sub(r"\(.*", "", name)


def full(path, traffic):
    hdr, units, rows = raw(path)
    idx = [(hdr.index(m), lab) for m, lab in METRICS if m in hdr]
    ki = hdr.index("Kernel Name")
    print(f"### ncu --set full (per launch) -- `{path.split('/')[-1]}`\n")
    print("| kernel | " + " | ".join(f"{lab} [{units[i]}]" for i, lab in idx) + " |")
    print("|---|" + "---|" * len(idx))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for r in rows:
        print(f"| `{short(r[ki])[:60]}` | " + " | ".join(r[i] for i, _ in idx) + " |")
        k = short(r[ki])
        if traffic is not None:  # summed over the captured launches of one kernel (one matvec / one assembly)
            g = lambda m: float(r[hdr.index(m)].replace(",", "")) * scale.get(units[hdr.index(m)], 1)
            ti = hdr.index("gpu__time_duration.sum")
            t = traffic.setdefault(k, {"time_us": 0.0, "dram_read_bytes": 0.0, "dram_write_bytes": 0.0, "launches": 0})
            t["time_us"] += float(r[ti].replace(",", "")) * UNITS.get(units[ti], 1.0) * 1e3
            t["dram_read_bytes"] += g("dram__bytes_read.sum")
            t["dram_write_bytes"] += g("dram__bytes_write.sum")
            t["launches"] += 1
    print()


if __name__ == "__main__":
    args = sys.argv[1:]
    tpath = None
    if "--traffic" in args:
        i = args.index("--traffic")
        tpath = args[i + 1]
        args = args[:i] + args[i + 2:]
    launches(args[0])
    traffic = {} if tpath else None
    for rep in args[1:]:
        full(rep, traffic)
    if tpath:
        json.dump({"source": "ncu --set full --clock-control none (tools/gpu_profile.sh, c2 step on B200); per launch, "
                             "summed over the captured launches of each kernel within one matvec (level-split graph: leaf-level + coarse far-field launches) or one assembly", "kernels": traffic}, open(tpath, "w"), indent=1)
