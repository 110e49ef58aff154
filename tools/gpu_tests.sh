#!/bin/bash
# the -m gpu suite (+ durations), output to gpurun_out/gputest.log
cd "$GRAFT_REPO_ROOT"
timeout 1500 python -m pytest tests -m gpu -q --durations=15 "$@" > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
