#!/bin/bash
# default bench (c5) + a short reference arm; outputs in gpurun_out/
cd "$GRAFT_REPO_ROOT"
tag=${1:-r02}
timeout 1500 python bench.py ${BENCH_ARGS:-} > gpurun_out/${tag}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${tag}_bench.log
if [ -n "$WITH_REF" ]; then
  timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${tag}_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/${tag}_ref.log
fi
