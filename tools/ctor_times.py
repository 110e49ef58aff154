"""H2Matrix constructor laps at a config (IGB_VERBOSE), cold then warm pool:
python tools/ctor_times.py c5 [device_partition]"""
import os
import sys
import time
os.environ["IGB_VERBOSE"] = "1"
sys.path.insert(0, ".")
import paper_1906_00785_b200 as igb
from bench import CONFIGS, make_disc
c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
dp = {"dp": True, "host": False}.get(sys.argv[2]) if len(sys.argv) > 2 else None
d = make_disc(igb, c)
for it in range(3):
    t = time.perf_counter()
    h = igb.H2Matrix(d, igb.H2Options(m=c["m"], eta=c["eta"]), device_partition=dp)
    print(f"ctor {it}: {time.perf_counter() - t:.3f} s", {k: round(v, 1) for k, v in h.assembly_times().items()},
          flush=True, file=sys.stderr)
    del h
