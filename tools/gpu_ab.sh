#!/bin/bash
# quick c2 timing (phase breakdown) + gpu test subset
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_golden.py -x -q -m gpu 2>&1 | tail -2
python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/ab.log 2>&1
python - << PY
import json
l=[x for x in open("gpurun_out/ab.log") if x.startswith("{")][-1]
d=json.loads(l); print("step", round(d["ms_per_step"],2), "asm", round(d["assembly_ms"],2), "mv", round(d["matvec_ms"],4), {k: round(v,4) for k,v in d["matvec_phase_ms"].items()})
PY
