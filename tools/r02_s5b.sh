#!/bin/bash
cd $GRAFT_REPO_ROOT
for cell in "0.6 0.6 8" "0.95 0.95 32"; do
  MMMCU_LIB=tools/_lib/csrsep.so timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    python tools/k1_profile.py $cell 3 > gpurun_out/s5b_k1_${cell// /_}.csv 2>/dev/null
done
python tools/k1csv.py gpurun_out/s5b_k1_*.csv
