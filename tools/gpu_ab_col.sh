#!/bin/bash
# far-field timing (c2, c5) of the current build + matvec dump for cross-build comparison
cd "$GRAFT_REPO_ROOT"
tag=${1:-cur}
timeout 300 python tools/ab_far_col.py $tag c2 c5 >> gpurun_out/ab_col.log 2>&1
