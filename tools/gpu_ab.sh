#!/bin/bash
# A/B the far-field kernel variants on c2 (phase times from bench.py)
mkdir -p gpurun_out
for v in 0 1 2 3; do
  IGB_FARSYM_VARIANT=$v python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/ab_$v.log 2>&1
  python - << PY
import json
l=[x for x in open("gpurun_out/ab_$v.log") if x.startswith("{")][-1]
d=json.loads(l); print("variant $v", "step", round(d["ms_per_step"],2), "mv", round(d["matvec_ms"],4), {k: round(v,4) for k,v in d["matvec_phase_ms"].items()})
PY
done
