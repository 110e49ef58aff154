#!/bin/bash
# singular-quadrature check: near-block parity tests + assembly kernel times (c2, c5, c3-space)
cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "near_blocks or matvec or far_field" > gpurun_out/sing_ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sing_ab_tests.log
python tools/asm_times.py 3 6 4 > gpurun_out/sing_ab_times.log 2>&1
python tools/asm_times.py 4 8 5 >> gpurun_out/sing_ab_times.log 2>&1
