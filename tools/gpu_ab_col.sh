#!/bin/bash
# A/B of far-field kernel variants: "<IGB_FAR_KERNEL> <MINB> <C>" triples as args
cd "$GRAFT_REPO_ROOT"
for v in "$@"; do
  set -- $v
  IGB_FAR_KERNEL=$1 IGB_FAR_COL_MINB=$2 IGB_FAR_COL_C=$3 timeout 300 python tools/ab_far_col.py $1$2$3 c2 c5 >> gpurun_out/ab_col.log 2>&1
done
