#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for o in 0 1 2; do IGB_NEAR_ORDER=$o timeout 300 python tools/ab_far_col.py order$o c2 c5 >> gpurun_out/ab_col.log 2>&1; done
