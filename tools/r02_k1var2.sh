#!/bin/bash
cd $GRAFT_REPO_ROOT
for n in prof r62p; do
  MMMCU_LIB=tools/_lib/$n.so timeout 300 python tools/k1_profile.py 0.6 0.6 8 4 > gpurun_out/v2_${n}.log 2>&1
  MMMCU_LIB=tools/_lib/$n.so timeout 300 python tools/k1_profile.py 0.9 0.9 16 4 >> gpurun_out/v2_${n}.log 2>&1
done
for n in base r62; do
  for cell in "0.6 0.6 8" "0.9 0.9 16"; do
    MMMCU_LIB=tools/_lib/$n.so timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"k1_" \
      python tools/k1_profile.py $cell 3 > gpurun_out/v2_${n}_${cell// /_}.csv 2>/dev/null
  done
done
