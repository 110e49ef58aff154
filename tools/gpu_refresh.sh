#!/bin/bash
# end-of-milestone evidence: tests, smoke, bench (both arms), launch list, ncu captures, full-size configs
bash tools/gpu_round.sh
PART=asm bash tools/gpu_profile.sh | tail -1
PART=mv bash tools/gpu_profile.sh | tail -1
for c in ${BIG:-c3 c4 c5}; do timeout 900 python tools/check_big.py $c > gpurun_out/big_$c.log 2>&1; tail -3 gpurun_out/big_$c.log; done
