#!/bin/bash
# A/B over values of one environment variable: tools/gpu_ab_env.sh VAR "<configs>" v1 v2 ...
cd "$GRAFT_REPO_ROOT"
var=$1; cfgs=$2; shift 2
for v in "$@"; do
  env $var=$v timeout 900 python tools/ab_far_col.py ${var}_$v $cfgs >> gpurun_out/ab_env.log 2>&1 || echo "$v failed" >> gpurun_out/ab_env.log
done
python - "$var" "$cfgs" "$@" >> gpurun_out/ab_env.log 2>&1 << 'PY'
import sys, numpy as np
var = sys.argv[1]; cfgs = sys.argv[2].split(); vals = sys.argv[3:]
for c in cfgs:
    y0 = np.load(f"gpurun_out/ab_{var}_{vals[0]}_{c}.npy")
    for v in vals[1:]:
        try:
            y = np.load(f"gpurun_out/ab_{var}_{v}_{c}.npy")
            print(f"{c}: |y({v}) - y({vals[0]})| / |y| = {np.linalg.norm(y - y0) / np.linalg.norm(y0):.3e}")
        except Exception as e:
            print(c, v, "missing", e)
PY
cat gpurun_out/ab_env.log
