"""per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the
matvec graph's kernels from an `ncu --set full` report, keyed by bench.py's
roofline names:  python tools/ncu_traffic.py report.ncu-rep out.json"""
import csv
import io
import json
import subprocess
import sys

ROLE = {"k_far_col_near": "far_leaf_near", "k_far_sym_near": "far_leaf_near", "k_far_col<": "far_coarse",
        "k_far_sym<": "far_coarse", "k_near_rows": "near_rows"}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

rep, out = sys.argv[1], sys.argv[2]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, units = rows[0], rows[1]
res = {}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    role = next((v for k, v in ROLE.items() if name.startswith("void " + k) or name.startswith(k)), None)
    if role is None:
        continue
    b = 0.0
    for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(key)
        b += float(r[i]) * UNIT.get(units[i], 1)
    res[role] = b
json.dump({"source": rep, "metric": "dram__bytes_read.sum + dram__bytes_write.sum per launch", "kernels": res},
          open(out, "w"), indent=1)
print(res)
