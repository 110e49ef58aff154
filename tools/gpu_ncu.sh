#!/bin/bash
# ncu --set full capture of selected kernels during one c2 step (1 GPU)
mkdir -p gpurun_out
KREGEX=${KREGEX:-"k_far_sym|k_near_rows|k_singular"}
NAME=${NAME:-prof}
python tools/profile_step.py c2 > gpurun_out/plain_${NAME}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${KREGEX}" -s 0 -c ${COUNT:-4} \
    -o gpurun_out/${NAME} python tools/profile_step.py c2 > gpurun_out/ncu_${NAME}.log 2>&1
echo "ncu rc=$?"
tail -2 gpurun_out/ncu_${NAME}.log
