#!/bin/bash
# singular DMMA check: P = 4 parity + c5 assembly times
cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_dense.py -q -m gpu -k "4-1-2-5 or P4 or laplace" > gpurun_out/dmma_tests.log 2>&1; echo "rc=$?" >> gpurun_out/dmma_tests.log
for v in 1 2; do python tools/asm_times.py 4 8 5 | sed "s/^/run=$v /" >> gpurun_out/dmma_times.log 2>&1; done
