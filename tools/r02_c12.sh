#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 60 python tools/tc_profile.py 0.6 0.6 8 5 > gpurun_out/c12_tc.log 2>&1 || exit 1
for cell in "0.6 0.95 32" "0.6 0.95 16" "0.6 0.9 32" "0.6 0.95 8" "0.6 0.8 32"; do
  timeout 60 python tools/tc_profile.py $cell 5 >> gpurun_out/c12_tc.log 2>&1
done
for n in s0 s4 base; do
  MMMCU_LIB=tools/_lib/$n.so timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k1_" \
      python tools/k1_profile.py 0.6 0.6 8 3 > gpurun_out/c12_k1_${n}.csv 2>/dev/null
done
