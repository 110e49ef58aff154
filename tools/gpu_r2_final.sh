#!/bin/bash
# round 2: GPU suite + default (c5) bench + reference arm + launch list + ncu of the dominant kernel
cd "$GRAFT_REPO_ROOT"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputest.log
timeout 1500 python bench.py > gpurun_out/r2_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/r2_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/r2_ref.log
# launch list: the first 400 launches of a c5 step (assembly + the first matvecs; cold-cache, serialised: shares, not absolutes)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_c5.csv \
    python tools/profile_step.py c5 > gpurun_out/r2_ncu_launch.log 2>&1; echo "launch rc=$?" >> gpurun_out/r2_ncu_launch.log
# the dominant kernel, full set
bash tools/gpu_ncu_src.sh r2_ws "^k_leaf_ws$" c5
