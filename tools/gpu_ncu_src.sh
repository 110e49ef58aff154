#!/bin/bash
# ncu --set full + source page (SASS with stall samples) of one kernel:
#   tools/gpu_ncu_src.sh <tag> <kernel regex> <config> [launch-skip]
cd "$GRAFT_REPO_ROOT"
tag=$1; rx=$2; cfg=${3:-c5}; skip=${4:-0}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -s $skip -c 1 -f -o gpurun_out/${tag} python tools/ncu_c5.py $cfg > gpurun_out/${tag}.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}.log
ncu -i gpurun_out/${tag}.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_sass.csv 2>> gpurun_out/${tag}.log
ncu -i gpurun_out/${tag}.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>> gpurun_out/${tag}.log
gzip -f gpurun_out/${tag}_sass.csv
rm -f gpurun_out/${tag}.ncu-rep
tail -3 gpurun_out/${tag}.log
