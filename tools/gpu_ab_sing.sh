#!/bin/bash
# A/B of compile-time variants of the singular kernel (NVFLAGS_EXTRA per variant)
cd paper_1906_00785_b200
for v in "$@"; do
  rm -f build/igb_device.o libigabem_b200.so
  make NVFLAGS_EXTRA="$v" -j4 > /dev/null 2>&1 || { echo "build failed: $v"; exit 1; }
  echo "variant: $v"
  (cd .. && python tools/asm_times.py)
done
