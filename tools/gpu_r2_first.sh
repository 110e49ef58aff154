#!/bin/bash
# round-2 first GPU call: GPU suite + a short c5 bench on the round-1 tree
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_smi.txt 2>&1
lscpu > gpurun_out/r2_lscpu.txt 2>&1; free -g >> gpurun_out/r2_lscpu.txt
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputest.log
timeout 900 python bench.py --config c5 --steps 2 --warmup 1 --no-cpu > gpurun_out/r2_bench_c5.log 2>&1; echo "bench rc=$?" >> gpurun_out/r2_bench_c5.log
