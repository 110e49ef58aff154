#!/bin/bash
# A/B of prebuilt library variants (ab/<name>/libigabem_b200.so, tools/build_variant.sh):
#   tools/gpu_ab_libs.sh "<configs>" base name1 name2 ...   ("base" = the in-tree build)
cd "$GRAFT_REPO_ROOT"
cfgs=$1; shift
for v in "$@"; do
  if [ "$v" = base ]; then unset IGB_B200_LIB; else export IGB_B200_LIB=$PWD/ab/$v/libigabem_b200.so; fi
  timeout 600 python tools/ab_far_col.py $v $cfgs >> gpurun_out/ab_libs.log 2>&1 || echo "$v failed" >> gpurun_out/ab_libs.log
done
python - "$cfgs" "$@" >> gpurun_out/ab_libs.log 2>&1 << 'PY'
import sys, numpy as np
cfgs = sys.argv[1].split(); names = sys.argv[2:]
for c in cfgs:
    y0 = np.load(f"gpurun_out/ab_{names[0]}_{c}.npy")
    for n in names[1:]:
        try:
            y = np.load(f"gpurun_out/ab_{n}_{c}.npy")
            print(f"{c}: |y_{n} - y_{names[0]}| / |y| = {np.linalg.norm(y - y0) / np.linalg.norm(y0):.3e}")
        except Exception as e:
            print(c, n, "missing", e)
PY
cat gpurun_out/ab_libs.log
