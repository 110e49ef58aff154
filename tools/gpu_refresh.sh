#!/bin/bash
# end-of-milestone evidence (two calls: gpurun copies back <= 64 MiB):
#   STAGE=1: tests, smoke, bench (both arms), launch list, ncu of the matvec kernels
#   STAGE=2: ncu of the assembly kernels, full-size configurations
if [ "${STAGE:-1}" = 1 ]; then
  bash tools/gpu_round.sh
  PART=mv bash tools/gpu_profile.sh | tail -1
else
  PART=asm bash tools/gpu_profile.sh | tail -1
  for c in ${BIG:-c3 c4 c5}; do timeout 900 python tools/check_big.py $c > gpurun_out/big_$c.log 2>&1; tail -3 gpurun_out/big_$c.log; done
fi
