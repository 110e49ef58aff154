#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_far_col -c 2 -o gpurun_out/r02_ncu_c5_far_col python tools/ncu_c5.py c5 > gpurun_out/r02_ncu_c5.log 2>&1
echo "rc=$?" >> gpurun_out/r02_ncu_c5.log
