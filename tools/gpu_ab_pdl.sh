#!/bin/bash
# A/B of programmatic dependent launch (IGB_PDL=1/0): single-GPU graph and per-rank dist matvecs
cd paper_1906_00785_b200
for v in "-DIGB_PDL=1" "-DIGB_PDL=0"; do
  rm -f build/igb_device.o libigabem_b200.so
  make NVFLAGS_EXTRA="$v" -j4 > /dev/null 2>&1 || { echo "build failed: $v"; exit 1; }
  echo "variant: $v"
  (cd .. && python tools/mv_times.py && python tools/dist_rank_time.py)
done
