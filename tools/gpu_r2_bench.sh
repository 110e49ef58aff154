#!/bin/bash
# round 2: GPU suite + default (c5) bench + reference arm
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputest.log
timeout 1500 python bench.py > gpurun_out/r2_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/r2_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/r2_ref.log
