#!/bin/bash
# ncu --set full of the c5 far-field kernels (the graph's own kernels)
cd "$GRAFT_REPO_ROOT"
tag=${1:-r02}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_far_col -c 2 -o gpurun_out/${tag}_ncu_c5_far python tools/ncu_c5.py c5 > gpurun_out/${tag}_ncu_c5.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_ncu_c5.log
