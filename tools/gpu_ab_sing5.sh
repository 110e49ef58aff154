#!/bin/bash
# A/B of singular-kernel variants on c5 (LapT<3>) assembly times
cd paper_1906_00785_b200
for v in "$@"; do
  rm -f build/igb_device.o libigabem_b200.so
  make NVFLAGS_EXTRA="$v" -j4 > /dev/null 2>&1 || { echo "build failed: $v"; exit 1; }
  echo "variant: $v"
  (cd .. && python tools/asm_times.py 4 8 5 | sed 's/.plan_host_ms.*regular_ms/ /')
done
