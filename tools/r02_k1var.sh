#!/bin/bash
cd $GRAFT_REPO_ROOT
for n in base noat nocompa nocompb stream; do
  for cell in "0.6 0.6 8" "0.9 0.9 16"; do
    MMMCU_LIB=tools/_lib/$n.so timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"k1_" \
      python tools/k1_profile.py $cell 4 > gpurun_out/r02_k1var_${n}_${cell// /_}.csv 2>/dev/null
  done
done
