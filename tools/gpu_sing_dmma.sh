#!/bin/bash
# DMMA A/B of the coincident singular accumulation (P = 4): parity + c5 assembly times
cd "$GRAFT_REPO_ROOT"
IGB_SING_DMMA=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -q -m gpu -k "4-1-2-5 or P4" > gpurun_out/dmma_tests.log 2>&1; echo "rc=$?" >> gpurun_out/dmma_tests.log
for v in 0 1 0 1; do IGB_SING_DMMA=$v python tools/asm_times.py 4 8 5 | sed "s/^/dmma=$v /" >> gpurun_out/dmma_times.log 2>&1; done
