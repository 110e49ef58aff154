#!/bin/bash
# launch list of one c2 step + full ncu capture of the far-field matvec and singular kernels
mkdir -p gpurun_out
python tools/profile_step.py c2 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
    python tools/profile_step.py c2 > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?"
python tools/profile_step.py c2 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_far|k_singular|k_near_leaf" -s 0 -c 6 \
    -o gpurun_out/prof_c2 python tools/profile_step.py c2 > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
tail -3 gpurun_out/ncu_full.log
