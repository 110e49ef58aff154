#!/bin/bash
# PART=launch: launch list of one c2 step; PART=asm / PART=mv: full ncu
# captures of the assembly / matvec kernels (separate calls: <= 64 MiB back)
mkdir -p gpurun_out
python tools/profile_step.py c2 > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
case "${PART:-launch}" in
launch)
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
      python tools/profile_step.py c2 > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?" ;;
asm)
  ncu --set full --clock-control none --import-source on -k regex:"k_singular|k_regular" -s 4 -c 4 \
      -o gpurun_out/prof_c2_asm -f python tools/profile_step.py c2 > gpurun_out/ncu_full_asm.log 2>&1; echo "asm rc=$?" ;;
mv)
  ncu --set full --clock-control none --import-source on \
      -k regex:"k_far_sym|k_near_rows|k_far_lower" -c 5 \
      -o gpurun_out/prof_c2_mv -f python tools/profile_step.py c2 > gpurun_out/ncu_full_mv.log 2>&1; echo "mv rc=$?" ;;
esac
