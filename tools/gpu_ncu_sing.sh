#!/bin/bash
# ncu --set full of the singular-quadrature kernels (one report per class),
# exported as raw CSV + per-source-line CSV on the box (reports stay there)
cd "$GRAFT_REPO_ROOT"
tag=${1:-r02}; cfg=${2:-c5}; classes=${3:-"0 1 2"}
mkdir -p /tmp/ncu
for k in $classes; do
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_singular --launch-skip $k -c 1 \
     -o /tmp/ncu/sing$k python tools/ncu_c5.py $cfg > gpurun_out/${tag}_ncu_sing$k.log 2>&1
  echo "rc=$?" >> gpurun_out/${tag}_ncu_sing$k.log
  ncu -i /tmp/ncu/sing$k.ncu-rep --page raw --csv > gpurun_out/${tag}_ncu_${cfg}_sing${k}_raw.csv 2>/dev/null
  ncu -i /tmp/ncu/sing$k.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_ncu_${cfg}_sing${k}_sass.csv 2>/dev/null
  gzip -f gpurun_out/${tag}_ncu_${cfg}_sing${k}_sass.csv
done
