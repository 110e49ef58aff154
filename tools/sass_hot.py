"""Hot spots from `ncu --page source --csv --print-source sass`: top instructions
by shared-memory wavefronts and by stall samples.  python tools/sass_hot.py file.csv[.gz] [n]"""
import csv
import gzip
import sys

path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
f = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
rows = list(csv.reader(f))
hdr = rows[1]
data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}


def num(r, k):
    try:
        return float(r[ix[k]])
    except (ValueError, KeyError):
        return 0.0


tot_wf = sum(num(r, "L1 Wavefronts Shared") for r in data)
tot_ex = sum(num(r, "L1 Wavefronts Shared Excessive") for r in data)
tot_s = sum(num(r, "Warp Stall Sampling (All Samples)") for r in data)
print(f"shared wavefronts {tot_wf:.3e} (excessive {tot_ex:.3e}); stall samples {tot_s:.0f}")
ops = {}
for r in data:
    op = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else "?"
    if op.startswith("@"):
        op = r[ix["Source"]].split()[1]
    op = op.split(".")[0]
    o = ops.setdefault(op, [0, 0, 0])
    o[0] += num(r, "Instructions Executed")
    o[1] += num(r, "Warp Stall Sampling (All Samples)")
    o[2] += num(r, "L1 Wavefronts Shared")
print("by opcode (warp insts, stall samples, shared wavefronts):")
for k, v in sorted(ops.items(), key=lambda kv: -kv[1][0])[:20]:
    print(f"  {k:10s} {v[0]:.3e} {v[1]:8.0f} {v[2]:.3e}")
print("top shared-wavefront instructions:")
for r in sorted(data, key=lambda r: -num(r, "L1 Wavefronts Shared"))[:n]:
    print(f"  {r[ix['Address']][-5:]} {r[ix['Source']].strip()[:60]:60s} wf {num(r, 'L1 Wavefronts Shared'):.2e} "
          f"ideal {num(r, 'L1 Wavefronts Shared Ideal'):.2e} exec {num(r, 'Instructions Executed'):.2e}")
